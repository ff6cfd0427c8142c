// common.cuh — internal declarations shared by the libarbor.so translation units.
// Not part of the C ABI (see include/arbor.h).
#pragma once

#include <cuda_runtime.h>
#include <cuda_bf16.h>
#include <stdint.h>

#include <string>
#include <utility>
#include <vector>

#include "../../include/arbor.h"

#define ARBOR_VERSION "arbor-b200 0.1.0 (sm_100a)"

namespace arbor {

constexpr int kAttnChunk = 64;       // slots per attention / score chunk
constexpr int kLeavesPerItem = 6;    // active leaves per attention work item (q rows staged)
constexpr size_t kInlineSeg = 256 * 1024;   // bytes of the inline plan segment
constexpr int kTileRecInts = 16;     // tensor-core tile record (build_plan): 2 halves + leaves[6]
constexpr int kStashSlots = 4;
constexpr int kQMaps = 4;            // cached q tensor maps (attn_tc.cu)
constexpr int kRingSlots = 32;
constexpr int kStageRing = 128;   // event pairs kept per profiled stage
constexpr size_t kRingBytes = 1u << 20;

// Error bits latched on the device (ctrl.err)
enum : int32_t {
  DERR_INVARIANT = 1,      // NaN / negative A, overflow
  DERR_OUT_OF_PAGES = 2,   // pool exhausted during append / rehydrate
  DERR_STATE = 4,
  DERR_INFEASIBLE = 8,     // device waterline raised Pressure on an infeasible budget
};

// Device-side control block (library-owned, one per context)
struct Ctrl {
  int32_t free_top;        // number of entries on the free stack
  int32_t err;             // DERR_* bits
  int32_t work_count;      // evict work items of the last plan
  int32_t rehyd_count;     // nodes rehydrated by the last plan
  int32_t plan_ticket;     // last-CTA ticket of the fused evict kernel (zero at rest)
  int32_t item_next;       // evict: next (node, row) work item to hand out (zero at rest)
  int32_t item_done;       // evict: select warps past the last item (zero at rest)
  int32_t gate;            // f1 device waterline: 1 when the last check raised Pressure
  int32_t pad_;
  long long pressure_events;   // Pressures raised by the device waterline
  long long evicted;       // tokens evicted by the last evict
  long long rehydrations;  // total rehydrations
  long long pages_in_use;  // pages held by nodes
};

// One evict work entry (a changed, non-pinned node): written by evict_plan, read by the
// select warps through 16-byte cp.async copies.
struct __align__(16) WorkEnt {
  int32_t node, kc, ka, n;   // node id, k_cur before, k_app after, n_i
  int64_t span;              // a_i (absolute position of the node's first token)
  int32_t foff;              // offset of its freed pages among all freed pages
  int16_t nfree, so;         // their count (≤ max_pages_node); soff before (< 2^15: int16 pos tags bound n)
};
constexpr int kEvictCtasPerSm = 2;
// CTAs of the side-stream PCIe copy kernels (stash / rehydrate, pages.cu): a small persistent
// grid — PCIe needs ~100 KB of reads in flight, not the whole GPU
constexpr int kCopyCtas = 32;
// decode_post / score_fused CTAs resident per SM (__launch_bounds__ min blocks): the score
// pass is split into parts only up to one resident wave
#ifndef ARBOR_POST_MINB
#define ARBOR_POST_MINB 2
#endif
constexpr int kPostCtasPerSm = ARBOR_POST_MINB;   // the fused evict kernel's work-list copies: [SMs·2][max_nodes]

// Valid slots of the chunk [c0, c0 + len) of a node's page list whose valid slots are
// [soff, soff + k_cur) (Q23*): [lo, hi) relative to c0, packed hi | lo << 8
// (len ≤ 255), 0 when the chunk holds none.
__host__ __device__ __forceinline__ int chunk_span(int soff, int kc, int c0, int len) {
  const int hi = min(len, max(0, soff + kc - c0));
  const int lo = min(len, max(0, soff - c0));
  return lo < hi ? (hi | (lo << 8)) : 0;
}
__host__ __device__ __forceinline__ int span_hi(int sp) { return sp & 255; }
__host__ __device__ __forceinline__ int span_lo(int sp) { return sp >> 8; }

// Per-launch geometry of the K/V pools
struct PoolGeom {
  int L, H, P, D, NP;   // local layers, local kv heads, page size, head dim, pages
  int max_pages_node;
};

struct DevState {
  int32_t *n, *kcur, *npages, *ptab, *free_stack;
  // soff: page-list slot of valid slot 0 (Q23*): the node's valid slots are
  // [soff, soff + k_cur) of its page list; entries below soff / P are freed (stale)
  int32_t *soff;
  int64_t *span;             // a_i
  int64_t *mass2;            // [2*max_nodes]: mass partial | mclose partial → all-reduced
  int64_t *mclose;           // this rank's Mclose partial
  int64_t *nq;               // Nq_i (uploaded)
  float *a, *s;              // last a_i, s_i
  float *ahat = nullptr;     // select_shared: slice-summed Â[t] (f32, by absolute position)
  Ctrl *ctrl;
  // tree mirror
  int32_t *parent, *len, *active;
  uint8_t *open, *onpath, *pinned;
  float *v, *u;
  int32_t *depth, *delta;
  double *Ed, *ED;
  // evict plan
  WorkEnt *work;             // changed non-pinned nodes of the last plan, ascending id
  // rehydrate / append plans
  int32_t *rehyd_nodes, *rehyd_flag;
  // attention / score plan (uploaded per call)
  int32_t *seg;              // packed plan when it exceeds the inline segment
  int32_t *inline_seg;       // packed plan, right after the tree mirror block (one H2D copy)
  float *partials;           // attention partials
  float *zbuf;               // attention log2-domain logits (fused score pass)
  int64_t *mass_part;        // this rank's per-node partial mass (cached, §score.cu)
  int64_t *mass_scratch;     // [max_nodes][layer_count] node-mass partials
  int64_t *mass_acc;         // [max_nodes] int64 accumulators of the fused score kernel (zero at rest)
  unsigned int *ticket;      // last-CTA ticket of the fused score kernel (zero at rest)
  unsigned int *row_done;    // [L·H] per-row tile counters of the tensor-core attention (zero at rest)
  long long *alloc_trace;    // debug builds only (ARBOR_ALLOC_TRACE)
  float *lse_scratch;        // used when arbor_score gets lse == NULL
  void *out_scratch;
};

// Plan of one attention / score call (built on the host from the tree, arbor_host.cu).
// A chunk is (node, kAttnChunk slots) of the union of the active leaves' paths; its pairs
// are the active leaves whose Path(ℓ_b) contains the node (pair p = ch_poff[c] + i), read
// once for all of them.  An attention item is a chunk with a subset of ≤ kLeavesPerItem of
// its leaves.  bp_list holds, per leaf b, its pairs in root→leaf, chunk-ascending order
// (the merge order).
// Thin slice 𝓛 × 𝓗 (arbor_params.slice_layers / slice_kv_heads) in this
// rank's local (layer, KV head) coordinates: rows l ≥ l_lo with h < h_hi.
struct SliceView {
  int l_lo, h_hi;
  __host__ __device__ bool has(int l, int h) const { return l >= l_lo && h < h_hi; }
};

struct PlanView {
  const int32_t *ch_node, *ch_chunk, *ch_poff, *ch_pcnt;   // C chunks: (node, chunk) + pairs
  const int4 *it_rec;                                       // I items: {node, c0, pair base, cnt}
  const int4 *tl_rec;                                       // T tensor-core tiles: {item A, item B|-1}
  const int32_t *pair_b;                                     // P pairs → active leaf index
  const int32_t *bp_off, *bp_list;                           // per leaf: pairs root→leaf
  int C, I, nA, P, T;
};

struct PoolView {
  int L, H, P, D, NP, MPN;    // local layers, kv heads, page size, head dim, pages, max pages/node
  int64_t max_tokens;
};

struct Snapshot {
  bool valid = false;
  int32_t *n, *kcur, *npages, *ptab, *free_stack, *soff;
  int64_t *mclose, *nq_dev, *mass_part;
  float *s;
  bool mass_valid = true;
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
  // CUDA Graph capture (arbor_capture_begin/end): main_stream is swapped for cap_stream while
  // capturing; uploads then go to pinned buffers owned by the graph, not the staging ring
  cudaStream_t cap_stream = nullptr, saved_ms = nullptr;
  bool capturing = false;
  std::vector<void *> cap_bufs;
  bool own_ms = false, own_ss = false;
  void *unc_part = nullptr, *unc_ticket = nullptr;   // f3 uncertainty scratch (grown on demand)
  size_t unc_cap = 0;
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
  long long geom_version = -1;   // tree_version whose geometry (a1) is on the device
  // staging ring
  void *ring[arbor::kRingSlots] = {};
  cudaEvent_t ring_ev[arbor::kRingSlots] = {};
  int ring_i = 0, ring_last = 0;
  // stash
  void *stash_host = nullptr;   // host pointer
  void *stash_dev = nullptr;    // device-visible pointer to the same memory
  bool own_stash = false;
  // rehydration: per-CTA staging of the retained rows that change slot (Q23r),
  // grown on demand
  void *rehyd_scratch = nullptr;
  size_t rehyd_scratch_bytes = 0;
  cudaEvent_t ev_main_to_side = nullptr, ev_side_done = nullptr;
  // lazy rehydration ("before the next decoding step"): the main stream waits for the
  // side-stream copy only when a call next reads or moves pool rows (attention, evict)
  cudaEvent_t ev_rehyd_done = nullptr, ev_stash_done = nullptr;
  bool rehyd_pending = false, stash_pending = false;
  std::vector<int32_t> rehyd_list;   // nodes of the pending rehydration copy
  bool side_pending = false;
  // attention scratch capacity
  size_t partial_cap = 0, seg_cap = 0, zbuf_cap = 0;
  // epoch: bumped by every call that changes KV contents / page tables
  long long epoch = 0, tree_version = 0;
  // logits of the last full-range tree_decode_attn (fused score pass)
  const void *lg_q = nullptr;
  const float *lg_lse = nullptr;
  long long lg_epoch = -1, lg_tree = -1;
  // cached per-node partial masses are exact for the current A (score.cu)
  bool mass_valid = true;
  int reduce_pending_n = -1;   // ARBOR_FLAG_EXTERNAL_REDUCE: N of the scores awaiting arbor_score_finish
  size_t scratch_q = 0;
  // NCCL
  void *nccl_comm = nullptr;
  void *nccl_lib = nullptr;
  // profiling
  cudaEvent_t st_ev[ARBOR_NUM_STAGES][arbor::kStageRing][2] = {};
  int st_count[ARBOR_NUM_STAGES] = {};   // launches recorded since the last reset
  bool st_created = false;
  bool profiling = true;                  // with ARBOR_FLAG_PROFILE: record stage events now
  long long launches = 0;
  arbor::Snapshot snap[arbor::kStashSlots];
  // tensor-core attention (attn_tc.cu): CUtensorMap storage for the K / V pools
  alignas(64) unsigned char tmap_k[128] = {};
  alignas(64) unsigned char tmap_v[128] = {};
  alignas(64) unsigned char tmap_k4[128] = {};  // 5-D views: 64-row boxes over consecutive pages
  alignas(64) unsigned char tmap_v4[128] = {};
  alignas(64) unsigned char tmap_q[arbor::kQMaps][128] = {};   // q maps of recent q buffers
  const void *tmap_q_ptr[arbor::kQMaps] = {};
  long long tmap_q_rows[arbor::kQMaps] = {};
  int tmap_q_box[arbor::kQMaps] = {};          // rows of the q box (query slot rows)
  int tmap_q_next = 0, tmap_q_cur = 0;
  bool tc_ok = false;
  int num_sms = 148;               // multiprocessors of the context's device
  const int64_t *nq_dev = nullptr;  // device Nq of the last score plan (inside the plan segment)
  std::string err;
};

// ---- launchers implemented in the kernel translation units ------------------------
namespace arbor {

// geometry.cu
void launch_geometry(arbor_ctx *c, int N, int nA);

// score.cu
void launch_node_mass(arbor_ctx *c, const int32_t *d_nodes, int num_nodes, int64_t *out,
                      int out_stride);
void launch_msve(arbor_ctx *c, int N, float *s_out);
// the thin slice in local coordinates, and the a_i normalisation |𝓛|·|𝓗_q| (Q4, Q6)
inline SliceView slice_view(const arbor_ctx *c) {
  const int lo_g = c->prm.slice_layers ? c->Lg - c->prm.slice_layers : 0;
  const int hi_g = c->prm.slice_kv_heads ? c->prm.slice_kv_heads : c->Hg;
  return SliceView{lo_g - c->cfg.layer_begin, hi_g - c->cfg.kv_head_begin};
}
inline double msve_norm(const arbor_ctx *c) {
  const double nl = c->prm.slice_layers ? c->prm.slice_layers : c->Lg;
  const double nh = c->prm.slice_kv_heads ? static_cast<double>(c->prm.slice_kv_heads) * c->G
                                          : static_cast<double>(c->Hqg);
  return nl * nh;
}
// nparts (a power of two) CTAs per (layer, KV head) row; CTA (row, p) owns the nodes with
// id & (nparts − 1) == p
void launch_score_fused(arbor_ctx *c, const PlanView &pv, const float *lse, const int32_t *d_nodes,
                        int num_nodes, int N, bool do_msve, float *s_out, int nparts);
// f2 (arbor_decode_step): merge of the attention partials (out, LSE) + the fused score of
// launch_score_fused in one launch; LSE stays on chip.  Requires decode_post_fits.
bool decode_post_fits(arbor_ctx *c, int nA);
void launch_decode_post(arbor_ctx *c, const PlanView &pv, void *out, float *lse_out,
                        const int32_t *d_nodes, int num_nodes, int N, bool do_msve, float *s_out,
                        int nparts);

// uncertainty.cu (f3)
arbor_status launch_uncertainty(arbor_ctx *c, const void *logits, int dtype, int batch, int vocab,
                                float *u_out);

// allocate.cu
// mode < 0: params.alloc_mode; only_node ≥ 0: targets of the other nodes are n (unchanged)
void launch_allocate(arbor_ctx *c, int N, int nA, const float *s, int64_t budget, int32_t *k_out,
                     int mode = -1, int only_node = -1, bool gated = false);
// f1 waterline (Alg. 2 l.31-33) on the device: ctrl->gate = (Σ_i k_cur_i ≥ thresh); a gated
// allocate then writes k_out = k_cur (no change) when the gate is 0.  infeasible: the
// budget cannot be met — a raised Pressure latches DERR_INFEASIBLE instead.
void launch_waterline(arbor_ctx *c, int N, int64_t thresh, bool infeasible);

// evict.cu
void launch_evict(arbor_ctx *c, int N, const int32_t *k_target, int max_n, bool gated = false);
// select_shared: Â[t] = Σ_{slice rows, ascending} A[l][h][t] in fp64, rounded to f32
void launch_ahat(arbor_ctx *c);

// pages.cu
void launch_append(arbor_ctx *c, int node, const void *k, const void *v, int n_old, int ntok);
void launch_stash(arbor_ctx *c, int node, int n, int64_t span);
void launch_rehydrate_plan(arbor_ctx *c, int count, int keep_floor);
void launch_rehydrate_copy(arbor_ctx *c, int count, int max_n);

// attn.cu
// returns true when the partials were also merged into out / lse (tensor-core path)
bool launch_attn_partial(arbor_ctx *c, const PlanView &pv, const void *q, int layer_begin,
                         int layer_count, int max_cnt, void *out, float *lse);
// attn_tc.cu (tcgen05 path for bf16, d = 128)
bool attn_tc_init(arbor_ctx *c);
bool launch_attn_tc(arbor_ctx *c, const PlanView &pv, const void *q, int layer_begin,
                    int layer_count, int max_cnt, void *out, float *lse);
void launch_attn_merge(arbor_ctx *c, const PlanView &pv, int layer_count, void *out,
                       float *lse);

void stage_begin(arbor_ctx *c, int st, cudaStream_t s);
void stage_end(arbor_ctx *c, int st, cudaStream_t s);

// Programmatic dependent launch: the kernel may start while the previous kernel on the stream
// drains (its prologue — smem carve-up, mbarrier init, TMEM alloc — overlaps that tail); every
// thread of a kernel launched this way calls pdl_wait() before it touches global memory the
// earlier kernels write or read.
template <typename... KArgs, typename... Args>
inline cudaError_t launch_pdl(void (*kernel)(KArgs...), dim3 grid, dim3 block, size_t smem,
                              cudaStream_t stream, Args &&...args) {
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = stream;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = at;
  static const int pdl_off = getenv("ARBOR_NO_PDL") ? 1 : 0;   // diagnostics
  cfg.numAttrs = pdl_off ? 0 : 1;
  return cudaLaunchKernelEx(&cfg, kernel, std::forward<Args>(args)...);
}

#ifdef __CUDACC__
// griddepcontrol.wait: all prerequisite grids complete and their memory visible (a no-op when
// the kernel was launched without the programmatic-serialization attribute)
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;\n" ::: "memory"); }
// griddepcontrol.launch_dependents: this CTA no longer holds back the next PDL-launched kernel
// (which launches once every CTA of this grid has triggered or exited, so all of this grid's
// CTAs are resident by then: no resource deadlock)
__device__ __forceinline__ void pdl_trigger() {
  asm volatile("griddepcontrol.launch_dependents;\n" ::: "memory");
}
#endif

}  // namespace arbor

#define ARBOR_LAUNCHED(c) ((c)->launches++)
