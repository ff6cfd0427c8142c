// common.cuh — internal declarations shared by the libarbor.so translation units.
// Not part of the C ABI (see include/arbor.h).
#pragma once

#include <cuda_runtime.h>
#include <cuda_bf16.h>
#include <stdint.h>

#include <string>
#include <vector>

#include "../../include/arbor.h"

#define ARBOR_VERSION "arbor-b200 0.1.0 (sm_100a)"

namespace arbor {

constexpr int kAttnChunk = 128;      // slots per attention / score segment
constexpr int kMaxQueriesPerCta = 64; // (leaves sharing a segment) x G per CTA
constexpr int kStashSlots = 4;
constexpr int kRingSlots = 8;
constexpr size_t kRingBytes = 4u << 20;

// Error bits latched on the device (ctrl.err)
enum : int32_t {
  DERR_INVARIANT = 1,      // NaN / negative A, overflow
  DERR_OUT_OF_PAGES = 2,   // pool exhausted during append / rehydrate
  DERR_STATE = 4,
};

// Device-side control block (library-owned, one per context)
struct Ctrl {
  int32_t free_top;        // number of entries on the free stack
  int32_t err;             // DERR_* bits
  int32_t work_count;      // evict work items of the last plan
  int32_t rehyd_count;     // nodes rehydrated by the last plan
  long long evicted;       // tokens evicted by the last evict
  long long rehydrations;  // total rehydrations
  long long pages_in_use;  // pages held by nodes
  long long pad;
};

// Per-launch geometry of the K/V pools
struct PoolGeom {
  int L, H, P, D, NP;   // local layers, local kv heads, page size, head dim, pages
  int max_pages_node;
};

struct DevState {
  int32_t *n, *kcur, *npages, *ptab, *free_stack;
  int64_t *span;             // a_i
  int64_t *mass2;            // [2*max_nodes]: mass partial | mclose partial → all-reduced
  int64_t *mclose;           // this rank's Mclose partial
  int64_t *nq;               // Nq_i (uploaded)
  float *a, *s;              // last a_i, s_i
  Ctrl *ctrl;
  // tree mirror
  int32_t *parent, *len, *active;
  uint8_t *open, *onpath, *pinned;
  float *v, *u;
  int32_t *depth, *delta;
  double *Ed, *ED;
  // evict plan
  int32_t *work_node, *work_old, *work_new;
  // rehydrate / append plans
  int32_t *rehyd_nodes, *rehyd_flag;
  // attention / score plan (uploaded per call)
  int32_t *seg;              // packed plan (see attn.cu)
  float *partials;           // attention partials
  float *lse_scratch;        // used when arbor_score gets lse == NULL
  void *out_scratch;
};

// Plan of one attention / score call (built on the host from the tree, arbor_host.cu).
// A segment is (node, chunk of kAttnChunk slots) of the union of the active leaves' paths;
// its leaf list names every active leaf whose Path(ℓ_b) contains the node (read once for
// all of them).  pair p = seg_loff[s] + i is the i-th leaf of segment s; bp_list holds,
// per leaf b, its pairs in root→leaf, chunk-ascending order (the merge order).
struct PlanView {
  const int32_t *seg_node, *seg_chunk, *seg_loff, *seg_lcnt, *pair_b, *bp_off, *bp_list;
  int S, nA, P;
};

struct PoolView {
  int L, H, P, D, NP, MPN;    // local layers, kv heads, page size, head dim, pages, max pages/node
  int64_t max_tokens;
};

struct Snapshot {
  bool valid = false;
  int32_t *n, *kcur, *npages, *ptab, *free_stack;
  int64_t *mclose, *nq_dev;
  float *s;
  Ctrl *ctrl;
  std::vector<int32_t> h_n;
  std::vector<uint8_t> h_open;
  std::vector<int64_t> h_span, h_nq;
  int num_known = 0;
};

}  // namespace arbor

struct arbor_ctx {
  arbor_config cfg;
  arbor_params prm;
  int L, H, Hq, G, D, P, NP, esize;
  int Lg, Hg, Hqg;
  int max_nodes, max_pages_node, max_active;
  int64_t max_tokens;
  cudaStream_t ms, ss;
  bool own_ms = false, own_ss = false;
  arbor::DevState d{};
  // host mirror
  std::vector<int32_t> h_n;
  std::vector<uint8_t> h_open;
  std::vector<int64_t> h_span, h_nq;
  int num_known = 0;
  // cached tree (to skip re-upload / geometry)
  std::vector<int32_t> t_parent, t_len, t_active;
  std::vector<uint8_t> t_open;
  std::vector<float> t_v, t_u;
  bool tree_valid = false;
  // staging ring
  void *ring[arbor::kRingSlots] = {};
  cudaEvent_t ring_ev[arbor::kRingSlots] = {};
  int ring_i = 0, ring_last = 0;
  // stash
  void *stash_host = nullptr;   // host pointer
  void *stash_dev = nullptr;    // device-visible pointer to the same memory
  bool own_stash = false;
  cudaEvent_t ev_main_to_side = nullptr, ev_side_done = nullptr;
  bool side_pending = false;
  // attention scratch capacity
  size_t partial_cap = 0, seg_cap = 0;
  // NCCL
  void *nccl_comm = nullptr;
  void *nccl_lib = nullptr;
  // profiling
  cudaEvent_t st_ev[ARBOR_NUM_STAGES][2] = {};
  bool st_used[ARBOR_NUM_STAGES] = {};
  long long launches = 0;
  arbor::Snapshot snap[arbor::kStashSlots];
  std::string err;
};

// ---- launchers implemented in the kernel translation units ------------------------
namespace arbor {

// geometry.cu
void launch_geometry(arbor_ctx *c, int N, int nA);

// score.cu
void launch_score_accum(arbor_ctx *c, const PlanView &pv, int max_q, const void *q,
                        const float *lse, int layer_count);
void launch_node_mass(arbor_ctx *c, const int32_t *d_nodes, int num_nodes, int64_t *out,
                      int out_stride);
void launch_msve(arbor_ctx *c, int N, float *s_out);

// allocate.cu
void launch_allocate(arbor_ctx *c, int N, const float *s, int64_t budget, int32_t *k_out);

// evict.cu
void launch_evict_plan(arbor_ctx *c, int N, const int32_t *k_target);
void launch_select_compact(arbor_ctx *c, int max_n);

// pages.cu
void launch_append(arbor_ctx *c, int node, const void *k, const void *v, int n_old, int ntok);
void launch_stash(arbor_ctx *c, int node, int n, int64_t span);
void launch_rehydrate_plan(arbor_ctx *c, int count);
void launch_rehydrate_copy(arbor_ctx *c, int count, int max_n);

// attn.cu
void launch_attn_partial(arbor_ctx *c, const PlanView &pv, int max_q, const void *q,
                         int layer_begin, int layer_count);
void launch_attn_merge(arbor_ctx *c, const PlanView &pv, int layer_count, void *out,
                       float *lse);

void stage_begin(arbor_ctx *c, int st, cudaStream_t s);
void stage_end(arbor_ctx *c, int st, cudaStream_t s);

}  // namespace arbor

#define ARBOR_LAUNCHED(c) ((c)->launches++)
