// arbor_host.cu — the C ABI of libarbor.so (include/arbor.h): argument and tree validation,
// host mirrors, launch planning and sequencing, stream/event management, NCCL bootstrap.
// Every step of the path runs in the kernels of geometry.cu, score.cu, allocate.cu,
// evict.cu, pages.cu and attn.cu; this file only validates, plans and enqueues.
#include <dlfcn.h>
#include <nccl.h>

#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <string>
#include <vector>

#include "common.cuh"

using namespace arbor;

namespace {

arbor_status fail(arbor_ctx *c, arbor_status s, const std::string &msg) {
  if (c) c->err = msg;
  return s;
}

#define CK(x)                                                                                  \
  do {                                                                                         \
    cudaError_t e_ = (x);                                                                      \
    if (e_ != cudaSuccess)                                                                     \
      return fail(c, ARBOR_ERR_CUDA, std::string(#x) + ": " + cudaGetErrorString(e_));         \
  } while (0)

#define CK_LAUNCH()                                                                            \
  do {                                                                                         \
    cudaError_t e_ = cudaGetLastError();                                                       \
    if (e_ != cudaSuccess)                                                                     \
      return fail(c, ARBOR_ERR_CUDA, std::string("kernel launch: ") + cudaGetErrorString(e_)); \
  } while (0)

// ---------------------------------------------------------------- NCCL (dlopen)
struct NcclApi {
  void *lib = nullptr;
  ncclResult_t (*getUniqueId)(ncclUniqueId *) = nullptr;
  ncclResult_t (*commInitRank)(ncclComm_t *, int, ncclUniqueId, int) = nullptr;
  ncclResult_t (*allReduce)(const void *, void *, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t,
                            cudaStream_t) = nullptr;
  ncclResult_t (*commDestroy)(ncclComm_t) = nullptr;
  const char *(*getErrorString)(ncclResult_t) = nullptr;
  bool load() {
    if (lib) return true;
    lib = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
    if (!lib) return false;
    getUniqueId = reinterpret_cast<decltype(getUniqueId)>(dlsym(lib, "ncclGetUniqueId"));
    commInitRank = reinterpret_cast<decltype(commInitRank)>(dlsym(lib, "ncclCommInitRank"));
    allReduce = reinterpret_cast<decltype(allReduce)>(dlsym(lib, "ncclAllReduce"));
    commDestroy = reinterpret_cast<decltype(commDestroy)>(dlsym(lib, "ncclCommDestroy"));
    getErrorString = reinterpret_cast<decltype(getErrorString)>(dlsym(lib, "ncclGetErrorString"));
    return getUniqueId && commInitRank && allReduce && commDestroy && getErrorString;
  }
};
NcclApi g_nccl;

// ---------------------------------------------------------------- helpers
template <typename T>
arbor_status dmalloc(arbor_ctx *c, T **p, size_t count) {
  if (count == 0) count = 1;
  CK(cudaMalloc(reinterpret_cast<void **>(p), count * sizeof(T)));
  CK(cudaMemsetAsync(*p, 0, count * sizeof(T), c->ms));
  return ARBOR_OK;
}

#define TRY(x)                                \
  do {                                        \
    arbor_status s_ = (x);                    \
    if (s_ != ARBOR_OK) return s_;            \
  } while (0)

// Pinned staging ring for host→device uploads: a slot is reused only after the copy that
// last read it has completed.
arbor_status ring_acquire(arbor_ctx *c, size_t bytes, void **out) {
  if (c->capturing) {
    // a captured copy reads its source at every replay: a pinned buffer owned by the graph
    CK(cudaHostAlloc(out, bytes > 0 ? bytes : 1, cudaHostAllocDefault));
    c->cap_bufs.push_back(*out);
    return ARBOR_OK;
  }
  if (bytes > kRingBytes) return fail(c, ARBOR_ERR_INVALID_ARG, "upload larger than staging ring");
  const int i = c->ring_i;
  CK(cudaEventSynchronize(c->ring_ev[i]));
  *out = c->ring[i];
  c->ring_i = (i + 1) % kRingSlots;
  c->ring_last = i;
  return ARBOR_OK;
}

arbor_status ring_upload(arbor_ctx *c, void *dst, const void *host_src, size_t bytes) {
  void *buf = nullptr;
  TRY(ring_acquire(c, bytes, &buf));
  std::memcpy(buf, host_src, bytes);
  CK(cudaMemcpyAsync(dst, buf, bytes, cudaMemcpyHostToDevice, c->ms));
  if (!c->capturing) CK(cudaEventRecord(c->ring_ev[c->ring_last], c->ms));
  return ARBOR_OK;
}

// ---------------------------------------------------------------- validation
arbor_status validate_params(const arbor_params *p, std::string &msg) {
  if (!p) { msg = "params is NULL"; return ARBOR_ERR_INVALID_ARG; }
  auto fin = [](double x) { return std::isfinite(x); };
  if (!fin(p->alpha) || p->alpha <= 0) { msg = "alpha must be > 0"; return ARBOR_ERR_INVALID_ARG; }
  if (!fin(p->gamma) || p->gamma < 0) { msg = "gamma must be >= 0"; return ARBOR_ERR_INVALID_ARG; }
  if (!fin(p->lambda_d) || !fin(p->lambda_delta)) { msg = "lambda must be finite"; return ARBOR_ERR_INVALID_ARG; }
  if (!fin(p->eta) || p->eta <= 0 || p->eta > 1) { msg = "eta must be in (0,1]"; return ARBOR_ERR_INVALID_ARG; }
  if (!fin(p->r_min) || p->r_min < 0 || p->r_min > 1) { msg = "r_min must be in [0,1]"; return ARBOR_ERR_INVALID_ARG; }
  if (p->k_min < 0 || p->l_tail < 0 || p->n_sinks < 0) { msg = "k_min, l_tail, n_sinks must be >= 0"; return ARBOR_ERR_INVALID_ARG; }
  if (p->alloc_mode < 0 || p->alloc_mode > 3) { msg = "bad alloc_mode"; return ARBOR_ERR_INVALID_ARG; }
  if (p->alloc_mode == ARBOR_ALLOC_STREAM && (p->l_tail != 0 || p->select_mode != ARBOR_SELECT_SINKS_TAIL)) {
    msg = "alloc_mode STREAM needs l_tail 0 and select_mode SINKS_TAIL"; return ARBOR_ERR_INVALID_ARG;
  }
  for (double t : p->theta) if (!fin(t)) { msg = "theta must be finite"; return ARBOR_ERR_INVALID_ARG; }
  if (p->select_mode < 0 || p->select_mode > 2) { msg = "bad select_mode"; return ARBOR_ERR_INVALID_ARG; }
  if (p->no_rehydrate != 0 && p->no_rehydrate != 1) { msg = "no_rehydrate must be 0 or 1"; return ARBOR_ERR_INVALID_ARG; }
  if (p->k_protect < 0) { msg = "k_protect must be >= 0"; return ARBOR_ERR_INVALID_ARG; }
  if (p->slice_layers < 0 || p->slice_kv_heads < 0) { msg = "slice sizes must be >= 0"; return ARBOR_ERR_INVALID_ARG; }
  if (p->select_shared != 0 && p->select_shared != 1) { msg = "select_shared must be 0 or 1"; return ARBOR_ERR_INVALID_ARG; }
  return ARBOR_OK;
}

arbor_status validate_tree_impl(const arbor_tree *t, int n_sinks, std::string &msg,
                                std::vector<int32_t> *depth_out = nullptr) {
  if (!t) { msg = "tree is NULL"; return ARBOR_ERR_INVALID_ARG; }
  const int N = t->num_nodes;
  if (N < 1) { msg = "tree needs at least the root"; return ARBOR_ERR_INVALID_ARG; }
  if (!t->parent || !t->span_start || !t->span_len || !t->is_open || !t->search_value ||
      !t->uncertainty) {
    msg = "tree array is NULL"; return ARBOR_ERR_INVALID_ARG;
  }
  if (t->num_active < 1 || !t->active) { msg = "need >= 1 active leaf"; return ARBOR_ERR_INVALID_ARG; }
  if (t->parent[0] != -1) { msg = "node 0 must be the root (parent -1)"; return ARBOR_ERR_INVALID_ARG; }
  std::vector<int32_t> depth(N, 0);
  for (int i = 0; i < N; ++i) {
    const int p = t->parent[i];
    if (i > 0 && (p < 0 || p >= i)) { msg = "parent id must satisfy 0 <= parent < child (node " + std::to_string(i) + ")"; return ARBOR_ERR_INVALID_ARG; }
    if (t->span_len[i] < 0 || t->span_start[i] < 0) { msg = "negative span"; return ARBOR_ERR_INVALID_ARG; }
    if (!t->is_open[i] && t->span_len[i] < 1) { msg = "closed node with n < 1"; return ARBOR_ERR_INVALID_ARG; }
    const float v = t->search_value[i], u = t->uncertainty[i];
    if (!(v >= 0.f && v <= 1.f) || !(u >= 0.f && u <= 1.f)) { msg = "v, u must lie in [0,1]"; return ARBOR_ERR_INVALID_ARG; }
    if (i > 0) {
      if (t->is_open[p]) { msg = "a node's parent must be closed"; return ARBOR_ERR_INVALID_ARG; }
      // spans along a root path do not overlap: a child starts after its parent ends
      if (t->span_start[i] < t->span_start[p] + t->span_len[p]) { msg = "child span overlaps its parent's"; return ARBOR_ERR_INVALID_ARG; }
      depth[i] = depth[p] + 1;
    }
  }
  std::vector<uint8_t> seen(N, 0);
  for (int b = 0; b < t->num_active; ++b) {
    const int a = t->active[b];
    if (a < 0 || a >= N) { msg = "active leaf is not a node"; return ARBOR_ERR_INVALID_ARG; }
    if (seen[a]) { msg = "duplicate active leaf"; return ARBOR_ERR_INVALID_ARG; }
    seen[a] = 1;
  }
  if (n_sinks > t->span_len[0]) { msg = "n_sinks > n_root"; return ARBOR_ERR_INVALID_ARG; }
  if (depth_out) *depth_out = std::move(depth);
  return ARBOR_OK;
}

// Path* (union of the active root paths, Q14)
std::vector<uint8_t> host_path_star(const arbor_tree *t) {
  std::vector<uint8_t> on(t->num_nodes, 0);
  for (int b = 0; b < t->num_active; ++b)
    for (int x = t->active[b]; x >= 0; x = t->parent[x]) on[x] = 1;
  return on;
}

// pinned (k = n, never evicted): open blocks, and Path* unless params.k_protect > 0
// or the flattened-stream analogue is the allocation (its path is a stream)
std::vector<uint8_t> host_pinned(const arbor_tree *t, const arbor_params *p) {
  const bool path_free = p->k_protect > 0 || p->alloc_mode == ARBOR_ALLOC_STREAM;
  std::vector<uint8_t> pin = path_free ? std::vector<uint8_t>(t->num_nodes, 0) : host_path_star(t);
  for (int i = 0; i < t->num_nodes; ++i) if (t->is_open[i]) pin[i] = 1;
  return pin;
}

int64_t floor_count_host(int n, const arbor_params *p) {
  const int tl = std::min(p->l_tail, n);
  const int64_t fr = static_cast<int64_t>(std::floor(p->r_min * static_cast<double>(n) + 1e-9));
  return std::min<int64_t>(n, std::max<int64_t>(std::max(p->k_min, tl), fr));
}

int64_t min_feasible(const arbor_params *p, const arbor_tree *t) {
  if (p->alloc_mode == ARBOR_ALLOC_STATIC) return 0;
  if (p->alloc_mode == ARBOR_ALLOC_STREAM) {   // open blocks + the root's sinks
    int64_t tot = t->is_open[0] ? 0 : std::min(p->n_sinks, t->span_len[0]);
    for (int i = 0; i < t->num_nodes; ++i) if (t->is_open[i]) tot += t->span_len[i];
    return tot;
  }
  const auto pin = host_pinned(t, p);
  const auto on = host_path_star(t);
  int64_t tot = 0;
  for (int i = 0; i < t->num_nodes; ++i) {
    const int n = t->span_len[i];
    int64_t f;
    if (pin[i]) f = n;
    else if (p->alloc_mode == ARBOR_ALLOC_WATERFILL) f = floor_count_host(n, p);
    else f = std::min(n, p->k_min);
    if (!pin[i] && on[i] && p->k_protect > 0) f = std::max<int64_t>(f, std::min(n, p->k_protect));
    tot += f;
  }
  return tot;
}

// The tree must describe exactly the nodes the library knows (spans, lengths, open flags).
arbor_status check_tree(arbor_ctx *c, const arbor_tree *t, std::vector<int32_t> *depth = nullptr) {
  std::string msg;
  arbor_status s = validate_tree_impl(t, c->prm.n_sinks, msg, depth);
  if (s != ARBOR_OK) return fail(c, s, msg);
  if (t->num_nodes != c->num_known)
    return fail(c, ARBOR_ERR_INVALID_ARG, "tree has " + std::to_string(t->num_nodes) +
                                              " nodes, the context knows " + std::to_string(c->num_known));
  if (t->num_active > c->max_active) return fail(c, ARBOR_ERR_INVALID_ARG, "too many active leaves");
  for (int i = 0; i < t->num_nodes; ++i) {
    if (t->span_start[i] != c->h_span[i] || t->span_len[i] != c->h_n[i] ||
        (t->is_open[i] != 0) != (c->h_open[i] != 0))
      return fail(c, ARBOR_ERR_INVALID_ARG, "tree node " + std::to_string(i) +
                                                " disagrees with the context (span / length / open)");
  }
  return ARBOR_OK;
}

// ---------------------------------------------------------------- tree upload (+ a1)
// the device tree mirror already holds this tree
static bool tree_same(const arbor_ctx *c, const arbor_tree *t) {
  const int N = t->num_nodes, nA = t->num_active;
  return c->tree_valid && static_cast<int>(c->t_parent.size()) == N &&
         static_cast<int>(c->t_active.size()) == nA &&
         std::memcmp(c->t_parent.data(), t->parent, N * 4) == 0 &&
         std::memcmp(c->t_len.data(), t->span_len, N * 4) == 0 &&
         std::memcmp(c->t_active.data(), t->active, nA * 4) == 0 &&
         std::memcmp(c->t_open.data(), t->is_open, N) == 0 &&
         std::memcmp(c->t_v.data(), t->search_value, N * 4) == 0 &&
         std::memcmp(c->t_u.data(), t->uncertainty, N * 4) == 0;
}

// bytes of the device tree mirror block [parent | len | active | v | u | open]
static size_t tree_block_bytes(const arbor_ctx *c) {
  return static_cast<size_t>(c->max_nodes) * 16 + static_cast<size_t>(c->max_active) * 4 +
         c->max_nodes;
}

// pack the tree with the device block's fixed offsets into host memory b
static void pack_tree(const arbor_ctx *c, const arbor_tree *t, char *b) {
  const int N = t->num_nodes, nA = t->num_active;
  const size_t MN = c->max_nodes, MA = c->max_active;
  std::memcpy(b, t->parent, N * 4);
  std::memcpy(b + MN * 4, t->span_len, N * 4);
  std::memcpy(b + MN * 8, t->active, nA * 4);
  std::memcpy(b + MN * 8 + MA * 4, t->search_value, N * 4);
  std::memcpy(b + MN * 12 + MA * 4, t->uncertainty, N * 4);
  std::memcpy(b + MN * 16 + MA * 4, t->is_open, N);
}

// host caches of the uploaded tree
static void tree_commit(arbor_ctx *c, const arbor_tree *t) {
  const int N = t->num_nodes, nA = t->num_active;
  c->t_parent.assign(t->parent, t->parent + N);
  c->t_len.assign(t->span_len, t->span_len + N);
  c->t_active.assign(t->active, t->active + nA);
  c->t_open.assign(t->is_open, t->is_open + N);
  c->t_v.assign(t->search_value, t->search_value + N);
  c->t_u.assign(t->uncertainty, t->uncertainty + N);
  c->tree_valid = true;
  ++c->tree_version;
}

arbor_status upload_tree(arbor_ctx *c, const arbor_tree *t) {
  if (tree_same(c, t)) return ARBOR_OK;
  const size_t bytes = tree_block_bytes(c);
  void *buf = nullptr;
  TRY(ring_acquire(c, bytes, &buf));
  pack_tree(c, t, static_cast<char *>(buf));
  CK(cudaMemcpyAsync(c->d.parent, buf, bytes, cudaMemcpyHostToDevice, c->ms));
  if (!c->capturing) CK(cudaEventRecord(c->ring_ev[c->ring_last], c->ms));
  // a1 runs inside arbor_allocate's kernel; arbor_evict launches it only if needed
  tree_commit(c, t);
  return ARBOR_OK;
}

// ---------------------------------------------------------------- attention / score plan
struct HostPlan {
  std::vector<int32_t> ch_node, ch_chunk, ch_poff, ch_pcnt, it_rec, pair_b, bp_off, bp_list;
  std::vector<int32_t> tl_rec;   // tensor-core tiles: kTileRecInts ints each (build_plan)
  int max_cnt = 0;               // most leaves in one item
  std::vector<std::vector<int32_t>> paths;
};

// tile_pairs: the tensor-core attention leaves one partial per (tile = chunks ch, ch+1 of a
// node, leaf), stored at the even chunk's pair — the merge lists then hold even chunks only;
// the CUDA-core kernel leaves one partial per chunk.
void build_plan(const arbor_tree *t, const std::vector<int32_t> &n_of, HostPlan &p,
                bool tile_pairs) {
  const int N = t->num_nodes, nA = t->num_active;
  std::vector<std::vector<int32_t>> leaves(N);
  p.paths.assign(nA, {});
  for (int b = 0; b < nA; ++b) {
    auto &path = p.paths[b];
    for (int x = t->active[b]; x >= 0; x = t->parent[x]) path.push_back(x);
    std::reverse(path.begin(), path.end());
    for (int x : path) leaves[x].push_back(b);
  }
  std::vector<int32_t> chunk_of(N, -1);
  struct SingleItem { int node, pair, cnt, j0; };
  std::vector<SingleItem> single;
  for (int x = 0; x < N; ++x) {
    if (leaves[x].empty()) continue;
    const int nch = (n_of[x] + kAttnChunk - 1) / kAttnChunk;
    if (nch == 0) continue;
    chunk_of[x] = static_cast<int32_t>(p.ch_node.size());
    const int lc = static_cast<int>(leaves[x].size());
    const int ng = (lc + kLeavesPerItem - 1) / kLeavesPerItem;
    p.max_cnt = std::max(p.max_cnt, std::min(kLeavesPerItem, lc));
    for (int ch = 0; ch < nch; ++ch) {
      const int c = static_cast<int>(p.ch_node.size());
      p.ch_node.push_back(x);
      p.ch_chunk.push_back(ch);
      p.ch_poff.push_back(static_cast<int32_t>(p.pair_b.size()));
      p.ch_pcnt.push_back(lc);
      p.pair_b.insert(p.pair_b.end(), leaves[x].begin(), leaves[x].end());
      for (int j0 = 0; j0 < lc; j0 += kLeavesPerItem) {   // {node, c0, pair base, cnt}
        p.it_rec.push_back(x);
        p.it_rec.push_back(ch * kAttnChunk);
        p.it_rec.push_back(p.ch_poff[c] + j0);
        p.it_rec.push_back(std::min(kLeavesPerItem, lc - j0));
      }
    }
    // tensor-core tiles, one self-contained record each (kTileRecInts ints, one load per tile
    // in the kernel): {node A, c0 A, pair A, cnt A, node B or -1, c0 B, pair B, cnt B,
    // leaves[6], 0, 0}.  A node of ≥ 2 chunks: chunks (ch, ch+1) of one leaf group (B shares
    // A's query columns: cnt B = 0).  Single-chunk items are packed two per tile below.
    const int cfirst = chunk_of[x];
    for (int gi = 0; gi < ng; ++gi) {
      const int j0 = gi * kLeavesPerItem, cnt = std::min(kLeavesPerItem, lc - j0);
      if (nch == 1) {
        single.push_back({x, p.ch_poff[cfirst] + j0, cnt, j0});
        continue;
      }
      for (int ch = 0; ch < nch; ch += 2) {
        const bool hb = ch + 1 < nch;
        const int32_t r[8] = {x, ch * kAttnChunk, p.ch_poff[cfirst + ch] + j0, cnt,
                              hb ? x : -1, (ch + 1) * kAttnChunk,
                              hb ? p.ch_poff[cfirst + ch + 1] + j0 : -1, 0};
        p.tl_rec.insert(p.tl_rec.end(), r, r + 8);
        for (int j = 0; j < kLeavesPerItem; ++j) p.tl_rec.push_back(j < cnt ? leaves[x][j0 + j] : 0);
        p.tl_rec.push_back(0);
        p.tl_rec.push_back(0);
      }
    }
  }
  // single-chunk items (short nodes, e.g. the open children of a DPTS frontier): two per tile,
  // one per 64-slot half, each half with its own query columns, as long as the pair's leaves
  // fit the plan's widest item (NQ unchanged)
  for (size_t i = 0; i < single.size();) {
    const SingleItem &u = single[i];
    const bool two = i + 1 < single.size() && u.cnt + single[i + 1].cnt <= p.max_cnt;
    const SingleItem &w = two ? single[i + 1] : u;
    const int32_t r[8] = {u.node, 0, u.pair, u.cnt, two ? w.node : -1, 0, two ? w.pair : -1,
                          two ? w.cnt : 0};
    p.tl_rec.insert(p.tl_rec.end(), r, r + 8);
    int nl = 0;
    for (int j = 0; j < u.cnt; ++j) p.tl_rec.push_back(leaves[u.node][u.j0 + j]), ++nl;
    if (two)
      for (int j = 0; j < w.cnt; ++j) p.tl_rec.push_back(leaves[w.node][w.j0 + j]), ++nl;
    for (; nl < kLeavesPerItem + 2; ++nl) p.tl_rec.push_back(0);
    i += two ? 2 : 1;
  }
  p.bp_off.assign(1, 0);
  for (int b = 0; b < nA; ++b) {
    for (int x : p.paths[b]) {
      if (chunk_of[x] < 0) continue;
      const int nch = (n_of[x] + kAttnChunk - 1) / kAttnChunk;
      const int pos = static_cast<int>(std::lower_bound(leaves[x].begin(), leaves[x].end(), b) -
                                       leaves[x].begin());
      for (int ch = 0; ch < nch; ch += tile_pairs ? 2 : 1)
        p.bp_list.push_back(p.ch_poff[chunk_of[x] + ch] + pos);
    }
    p.bp_off.push_back(static_cast<int32_t>(p.bp_list.size()));
  }
}

// Upload [plan arrays | extra int32 list] (+ Nq when with_nq); fill a PlanView.  With a
// tree t, the tree mirror is (re)uploaded too — in the SAME copy when the plan fits the
// inline segment that follows the tree block on the device (every H2D copy on the stream
// costs ~4 µs of device time: C2 step 220 → 216 µs for one copy fewer, A/B).
arbor_status upload_plan(arbor_ctx *c, const HostPlan &p, int nA, bool with_nq,
                         const std::vector<int32_t> *extra, PlanView &pv, const int32_t **d_extra,
                         const arbor_tree *t = nullptr) {
  std::vector<int32_t> packed;
  auto put = [&](const std::vector<int32_t> &v) {
    const size_t off = packed.size();
    packed.insert(packed.end(), v.begin(), v.end());
    return off;
  };
  const size_t o_ir = put(p.it_rec);   // first: 16-byte aligned int4 records
  const size_t o_tl = put(p.tl_rec);   // int4 records (it_rec has 4 ints per item)
  const size_t o_cn = put(p.ch_node), o_cc = put(p.ch_chunk), o_cpo = put(p.ch_poff),
               o_cpc = put(p.ch_pcnt), o_pb = put(p.pair_b), o_bpo = put(p.bp_off),
               o_bpl = put(p.bp_list);
  const size_t o_extra = packed.size();
  if (extra) put(*extra);
  // Nq (int64, 8-byte aligned) rides in the same copy: one cudaMemcpyAsync per call
  if (packed.size() & 1) packed.push_back(0);
  const size_t o_nq = packed.size();
  static const bool split_nq = getenv("ARBOR_SPLIT_NQ") != nullptr;   // A/B: separate copy
  if (with_nq && split_nq) {
    TRY(ring_upload(c, c->d.nq, c->h_nq.data(), c->num_known * sizeof(int64_t)));
    c->nq_dev = c->d.nq;
  } else if (with_nq) {
    packed.resize(o_nq + 2 * static_cast<size_t>(c->num_known));
    std::memcpy(packed.data() + o_nq, c->h_nq.data(), c->num_known * sizeof(int64_t));
  }
  const size_t plan_bytes = packed.size() * 4;
  const int32_t *base = nullptr;
  const bool tree_new = t && !tree_same(c, t);
  if (plan_bytes <= kInlineSeg) {
    base = c->d.inline_seg;
    if (tree_new) {   // one copy: [tree block | pad | plan] → [d.parent … inline_seg]
      const size_t off = reinterpret_cast<const char *>(c->d.inline_seg) -
                         reinterpret_cast<const char *>(c->d.parent);
      void *buf = nullptr;
      TRY(ring_acquire(c, off + plan_bytes, &buf));
      pack_tree(c, t, static_cast<char *>(buf));
      if (plan_bytes) std::memcpy(static_cast<char *>(buf) + off, packed.data(), plan_bytes);
      CK(cudaMemcpyAsync(c->d.parent, buf, off + plan_bytes, cudaMemcpyHostToDevice, c->ms));
      if (!c->capturing) CK(cudaEventRecord(c->ring_ev[c->ring_last], c->ms));
      tree_commit(c, t);
    } else if (!packed.empty()) {
      TRY(ring_upload(c, c->d.inline_seg, packed.data(), plan_bytes));
    }
  } else {
    if (tree_new) TRY(upload_tree(c, t));
    if (plan_bytes > c->seg_cap) {
      if (c->d.seg) CK(cudaFree(c->d.seg));
      c->seg_cap = std::max<size_t>(plan_bytes * 2, 1 << 16);
      CK(cudaMalloc(&c->d.seg, c->seg_cap));
    }
    TRY(ring_upload(c, c->d.seg, packed.data(), plan_bytes));
    base = c->d.seg;
  }
  if (with_nq && !split_nq) c->nq_dev = reinterpret_cast<const int64_t *>(base + o_nq);
  pv.ch_node = base + o_cn;
  pv.ch_chunk = base + o_cc;
  pv.ch_poff = base + o_cpo;
  pv.ch_pcnt = base + o_cpc;
  pv.it_rec = reinterpret_cast<const int4 *>(base + o_ir);
  pv.tl_rec = reinterpret_cast<const int4 *>(base + o_tl);
  pv.T = static_cast<int>(p.tl_rec.size() / kTileRecInts);
  pv.pair_b = base + o_pb;
  pv.bp_off = base + o_bpo;
  pv.bp_list = base + o_bpl;
  pv.C = static_cast<int>(p.ch_node.size());
  pv.I = static_cast<int>(p.it_rec.size() / 4);
  pv.nA = nA;
  pv.P = static_cast<int>(p.pair_b.size());
  if (d_extra) *d_extra = base + o_extra;
  return ARBOR_OK;
}

arbor_status ensure_partials(arbor_ctx *c, size_t pairs, int layer_count) {
  const size_t need = pairs * layer_count * c->Hq * (c->D + 2) * sizeof(float);
  const size_t zneed = pairs * layer_count * c->Hq * kAttnChunk * sizeof(float);
  if (need > c->partial_cap) {
    if (c->d.partials) CK(cudaFree(c->d.partials));
    c->partial_cap = std::max<size_t>(need + need / 2, 1 << 20);
    CK(cudaMalloc(&c->d.partials, c->partial_cap));
  }
  if (zneed > c->zbuf_cap) {
    if (c->d.zbuf) CK(cudaFree(c->d.zbuf));
    c->zbuf_cap = std::max<size_t>(zneed + zneed / 2, 1 << 20);
    CK(cudaMalloc(&c->d.zbuf, c->zbuf_cap));
  }
  return ARBOR_OK;
}

void wait_rehydrated(arbor_ctx *c);

arbor_status run_attention(arbor_ctx *c, const HostPlan &hp, const PlanView &pv, int layer_begin,
                           int layer_count, const void *q, void *out, float *lse) {
  TRY(ensure_partials(c, hp.pair_b.size(), layer_count));
  wait_rehydrated(c);
  const bool merged = launch_attn_partial(c, pv, q, layer_begin, layer_count, hp.max_cnt, out, lse);
  CK_LAUNCH();
  if (!merged) {
    launch_attn_merge(c, pv, layer_count, out, lse);
    CK_LAUNCH();
  }
  return ARBOR_OK;
}

void wait_side(arbor_ctx *c) {
  if (c->side_pending) {
    cudaStreamWaitEvent(c->ms, c->ev_side_done, 0);
  }
  c->rehyd_pending = false;   // ev_side_done follows every side-stream copy
  c->stash_pending = false;
}

// pending write-through stash copies read the pages of their (closed) nodes
void wait_stash(arbor_ctx *c) {
  if (c->stash_pending) {
    cudaStreamWaitEvent(c->ms, c->ev_stash_done, 0);
    c->stash_pending = false;
  }
}

// before a launch that reads pool rows restored by a pending rehydration (the attention)
void wait_rehydrated(arbor_ctx *c) {
  if (c->rehyd_pending) {
    cudaStreamWaitEvent(c->ms, c->ev_rehyd_done, 0);
    c->rehyd_pending = false;
    c->rehyd_list.clear();
  }
}

arbor_status latched(arbor_ctx *c) {
  Ctrl h{};
  CK(cudaMemcpy(&h, c->d.ctrl, sizeof(Ctrl), cudaMemcpyDeviceToHost));
  if (h.err) {
    const int32_t zero = 0;
    CK(cudaMemcpy(&c->d.ctrl->err, &zero, sizeof(zero), cudaMemcpyHostToDevice));
    if (h.err & DERR_INVARIANT)
      return fail(c, ARBOR_ERR_INVARIANT, "device: invalid accumulated attention / weight (NaN, negative or out of range)");
    if (h.err & DERR_OUT_OF_PAGES) return fail(c, ARBOR_ERR_OUT_OF_PAGES, "device: page pool exhausted");
    if (h.err & DERR_INFEASIBLE) return fail(c, ARBOR_ERR_INFEASIBLE_BUDGET, "device waterline: Pressure on an infeasible budget");
    return fail(c, ARBOR_ERR_STATE, "device: state error");
  }
  return ARBOR_OK;
}

arbor_status sync_all(arbor_ctx *c) {
  CK(cudaStreamSynchronize(c->ss));
  CK(cudaStreamSynchronize(c->ms));
  return latched(c);
}

__global__ void init_node_kernel(int node, int64_t span, int32_t *n, int32_t *kcur, int32_t *npages,
                                 int32_t *soff, int64_t *span_arr, int64_t *mclose, float *s,
                                 float *a) {
  n[node] = 0;
  kcur[node] = 0;
  npages[node] = 0;
  soff[node] = 0;
  span_arr[node] = span;
  mclose[node] = 0;
  s[node] = 0.5f;
  a[node] = 0.f;
}

__global__ void init_free_kernel(int32_t *free_stack, int num_pages, Ctrl *ctrl) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < num_pages) free_stack[i] = num_pages - 1 - i;   // pops yield 0, 1, 2, …
  if (i == 0) {
    ctrl->free_top = num_pages;
    ctrl->err = 0;
    ctrl->work_count = 0;
    ctrl->rehyd_count = 0;
    ctrl->evicted = 0;
    ctrl->rehydrations = 0;
    ctrl->pages_in_use = 0;
    ctrl->gate = 0;
    ctrl->pressure_events = 0;
    ctrl->item_next = 0;
    ctrl->item_done = 0;
    ctrl->plan_ticket = 0;
  }
}

__global__ void fill_f32(float *p, int n, float v) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) p[i] = v;
}

}  // namespace

// ---------------------------------------------------------------- profiling hooks
namespace arbor {
// Profiling: every stage launch is bracketed by a pair of CUDA events on its stream; the
// last kStageRing pairs per stage are kept and averaged by arbor_stage_times (no sync here).
void stage_begin(arbor_ctx *c, int st, cudaStream_t s) {
  if ((c->cfg.flags & ARBOR_FLAG_PROFILE) && c->profiling)
    cudaEventRecord(c->st_ev[st][c->st_count[st] % kStageRing][0], s);
}
void stage_end(arbor_ctx *c, int st, cudaStream_t s) {
  if ((c->cfg.flags & ARBOR_FLAG_PROFILE) && c->profiling) {
    cudaEventRecord(c->st_ev[st][c->st_count[st] % kStageRing][1], s);
    ++c->st_count[st];
  }
}
}  // namespace arbor

// ================================================================ C ABI
extern "C" {

const char *arbor_version(void) { return ARBOR_VERSION; }

const char *arbor_status_string(arbor_status s) {
  switch (s) {
    case ARBOR_OK: return "ok";
    case ARBOR_ERR_INVALID_ARG: return "invalid argument";
    case ARBOR_ERR_INFEASIBLE_BUDGET: return "infeasible budget";
    case ARBOR_ERR_INVARIANT: return "invariant violated";
    case ARBOR_ERR_IO: return "host stash I/O error";
    case ARBOR_ERR_OUT_OF_PAGES: return "out of pages";
    case ARBOR_ERR_STATE: return "lifecycle state error";
    case ARBOR_ERR_CUDA: return "CUDA error";
    case ARBOR_ERR_NCCL: return "NCCL error";
  }
  return "unknown status";
}

const char *arbor_last_error(const arbor_ctx *ctx) { return ctx ? ctx->err.c_str() : ""; }

arbor_status arbor_validate_tree(const arbor_tree *tree, int32_t n_sinks, char *msg, size_t msg_len) {
  std::string m;
  arbor_status s = validate_tree_impl(tree, n_sinks, m);
  if (msg && msg_len) {
    std::snprintf(msg, msg_len, "%s", m.c_str());
  }
  return s;
}

arbor_status arbor_min_feasible_budget(const arbor_params *params, const arbor_tree *tree,
                                       int64_t *out) {
  std::string m;
  arbor_status s = validate_params(params, m);
  if (s != ARBOR_OK) return s;
  s = validate_tree_impl(tree, params->n_sinks, m);
  if (s != ARBOR_OK) return s;
  if (!out) return ARBOR_ERR_INVALID_ARG;
  *out = min_feasible(params, tree);
  return ARBOR_OK;
}

arbor_status arbor_nccl_unique_id(void *out128) {
  if (!out128) return ARBOR_ERR_INVALID_ARG;
  if (!g_nccl.load()) return ARBOR_ERR_NCCL;
  ncclUniqueId id;
  if (g_nccl.getUniqueId(&id) != ncclSuccess) return ARBOR_ERR_NCCL;
  std::memcpy(out128, &id, sizeof(id));
  return ARBOR_OK;
}

arbor_status arbor_init(const arbor_config *cfg, const arbor_params *params, arbor_ctx **out) {
  if (!out) return ARBOR_ERR_INVALID_ARG;
  *out = nullptr;
  if (!cfg) return ARBOR_ERR_INVALID_ARG;
  std::string msg;
  if (validate_params(params, msg) != ARBOR_OK) return ARBOR_ERR_INVALID_ARG;
  const arbor_config &k = *cfg;
  if (k.num_layers < 1 || k.num_kv_heads < 1 || k.num_q_heads < 1 || k.num_q_heads % k.num_kv_heads)
    return ARBOR_ERR_INVALID_ARG;
  if (k.head_dim != 64 && k.head_dim != 128) return ARBOR_ERR_INVALID_ARG;
  if (k.layer_begin < 0 || k.layer_count < 1 || k.layer_begin + k.layer_count > k.num_layers)
    return ARBOR_ERR_INVALID_ARG;
  if (k.kv_head_begin < 0 || k.kv_head_count < 1 || k.kv_head_begin + k.kv_head_count > k.num_kv_heads)
    return ARBOR_ERR_INVALID_ARG;
  if (k.kv_dtype != ARBOR_F32 && k.kv_dtype != ARBOR_BF16) return ARBOR_ERR_INVALID_ARG;
  if (k.page_size < 2 || k.page_size > 1024 || (k.page_size & (k.page_size - 1)) || k.num_pages < 1)
    return ARBOR_ERR_INVALID_ARG;   // page size: a power of two (shift addressing)
  if (k.max_nodes < 1 || k.max_nodes > 3072) return ARBOR_ERR_INVALID_ARG;   // a4 smem
  if (k.max_node_tokens < 1 || k.max_node_tokens > 32767) return ARBOR_ERR_INVALID_ARG;
  if (k.max_active < 1 || k.max_active > 1024 || k.max_tokens < 1) return ARBOR_ERR_INVALID_ARG;
  if (!k.k_pool || !k.v_pool || !k.pos_pool || !k.score) return ARBOR_ERR_INVALID_ARG;
  if (k.world_size < 1 || k.rank < 0 || k.rank >= k.world_size) return ARBOR_ERR_INVALID_ARG;
  const bool ext_reduce = (k.flags & ARBOR_FLAG_EXTERNAL_REDUCE) != 0;
  const bool coll = (k.flags & ARBOR_FLAG_COLLECTIVE) != 0;
  if ((k.world_size > 1 || coll) && !k.nccl_unique_id && !ext_reduce) return ARBOR_ERR_INVALID_ARG;
  if (coll && ext_reduce) return ARBOR_ERR_INVALID_ARG;
  if (params->slice_layers > k.num_layers || params->slice_kv_heads > k.num_kv_heads)
    return ARBOR_ERR_INVALID_ARG;
  if (params->select_shared && k.world_size > 1) return ARBOR_ERR_INVALID_ARG;   // Â is rank-local

  arbor_ctx *c = new arbor_ctx();
  c->cfg = k;
  c->prm = *params;
  c->L = k.layer_count;
  c->H = k.kv_head_count;
  c->G = k.num_q_heads / k.num_kv_heads;
  c->Hq = c->H * c->G;
  c->D = k.head_dim;
  c->P = k.page_size;
  c->NP = k.num_pages;
  c->esize = k.kv_dtype == ARBOR_BF16 ? 2 : 4;
  c->Lg = k.num_layers;
  c->Hg = k.num_kv_heads;
  c->Hqg = k.num_q_heads;
  c->max_nodes = k.max_nodes;
  c->max_pages_node = (k.max_node_tokens + k.page_size - 1) / k.page_size;
  c->max_active = k.max_active;
  c->max_tokens = k.max_tokens;
  auto bail = [&](arbor_status s) { arbor_destroy(c); return s; };
  // main_stream is used as given: NULL is the legacy default stream (a valid cudaStream_t)
  c->ms = static_cast<cudaStream_t>(k.main_stream);
  if (k.side_stream) c->ss = static_cast<cudaStream_t>(k.side_stream);
  else { if (cudaStreamCreateWithFlags(&c->ss, cudaStreamNonBlocking) != cudaSuccess) return bail(ARBOR_ERR_CUDA); c->own_ss = true; }

  const int MN = c->max_nodes, MA = c->max_active;
  DevState &d = c->d;
  arbor_status s = ARBOR_OK;
#define ALLOC(ptr, cnt) do { s = dmalloc(c, &(ptr), (cnt)); if (s != ARBOR_OK) return bail(s); } while (0)
  ALLOC(d.n, MN); ALLOC(d.kcur, MN); ALLOC(d.npages, MN); ALLOC(d.soff, MN);
  ALLOC(d.ptab, static_cast<size_t>(MN) * c->max_pages_node);
  ALLOC(d.free_stack, c->NP);
  ALLOC(d.span, MN); ALLOC(d.mass2, 2 * MN); ALLOC(d.mclose, MN); ALLOC(d.nq, MN);
  ALLOC(d.a, MN); ALLOC(d.s, MN); ALLOC(d.mass_part, MN);
  ALLOC(d.mass_scratch, static_cast<size_t>(MN) * c->L);
  ALLOC(d.mass_acc, MN);
  ALLOC(d.ticket, 1);
  ALLOC(d.row_done, static_cast<size_t>(c->L) * c->H);
  ALLOC(d.ctrl, 1);
  {
    // tree mirror block: [parent | len | active | v | u | open] (fixed offsets, see upload_tree)
    // followed (16-byte aligned) by the inline plan segment (upload_plan: one copy for both)
    char *blk = nullptr;
    const size_t tb = (static_cast<size_t>(MN) * 16 + static_cast<size_t>(MA) * 4 + MN + 255) & ~size_t(255);
    const size_t bytes = tb + kInlineSeg;
    if (cudaMalloc(&blk, bytes) != cudaSuccess) return bail(ARBOR_ERR_CUDA);
    d.inline_seg = reinterpret_cast<int32_t *>(blk + tb);
    d.parent = reinterpret_cast<int32_t *>(blk);
    d.len = reinterpret_cast<int32_t *>(blk + MN * 4);
    d.active = reinterpret_cast<int32_t *>(blk + MN * 8);
    d.v = reinterpret_cast<float *>(blk + MN * 8 + MA * 4);
    d.u = reinterpret_cast<float *>(blk + MN * 12 + MA * 4);
    d.open = reinterpret_cast<uint8_t *>(blk + MN * 16 + MA * 4);
  }
  ALLOC(d.onpath, MN); ALLOC(d.pinned, MN); ALLOC(d.depth, MN); ALLOC(d.delta, MN);
  ALLOC(d.Ed, 2 * MN + 2); ALLOC(d.ED, 2 * MN + 2);
  {
    int sms = 148;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    c->num_sms = sms;
    ALLOC(d.work, static_cast<size_t>(sms) * kEvictCtasPerSm * MN);
  }
  {
    // compaction rows are addressed with int32 row ids
    const int64_t rows_total = static_cast<int64_t>(c->L) * c->NP * c->H * c->P;
    if (rows_total >= (1ll << 31)) { c->err = "pool too large for int32 row ids"; return bail(ARBOR_ERR_INVALID_ARG); }
  }
  ALLOC(d.rehyd_nodes, MN + 1); ALLOC(d.rehyd_flag, MN + 2);
  if (params->select_shared) ALLOC(d.ahat, static_cast<size_t>(k.max_tokens));
#undef ALLOC
  init_free_kernel<<<(c->NP + 255) / 256, 256, 0, c->ms>>>(d.free_stack, c->NP, d.ctrl);
  fill_f32<<<(MN + 255) / 256, 256, 0, c->ms>>>(d.s, MN, 0.5f);
  c->launches += 2;
  {
    // E_d[x] = e^{−λ_d x}, E_Δ[x] = e^{−λ_Δ x} from host libm (Q9)
    std::vector<double> Ed(2 * MN + 2), ED(2 * MN + 2);
    for (int x = 0; x < 2 * MN + 2; ++x) {
      Ed[x] = std::exp(-params->lambda_d * x);
      ED[x] = std::exp(-params->lambda_delta * x);
    }
    if (cudaMemcpy(d.Ed, Ed.data(), Ed.size() * 8, cudaMemcpyHostToDevice) != cudaSuccess ||
        cudaMemcpy(d.ED, ED.data(), ED.size() * 8, cudaMemcpyHostToDevice) != cudaSuccess)
      return bail(ARBOR_ERR_CUDA);
  }
  for (int i = 0; i < kRingSlots; ++i) {
    if (cudaHostAlloc(&c->ring[i], kRingBytes, cudaHostAllocDefault) != cudaSuccess) return bail(ARBOR_ERR_CUDA);
    if (cudaEventCreateWithFlags(&c->ring_ev[i], cudaEventDisableTiming) != cudaSuccess) return bail(ARBOR_ERR_CUDA);
    cudaEventRecord(c->ring_ev[i], c->ms);
  }
  if (cudaEventCreateWithFlags(&c->ev_main_to_side, cudaEventDisableTiming) != cudaSuccess ||
      cudaEventCreateWithFlags(&c->ev_side_done, cudaEventDisableTiming) != cudaSuccess ||
      cudaEventCreateWithFlags(&c->ev_rehyd_done, cudaEventDisableTiming) != cudaSuccess ||
      cudaEventCreateWithFlags(&c->ev_stash_done, cudaEventDisableTiming) != cudaSuccess)
    return bail(ARBOR_ERR_CUDA);
  if (k.flags & ARBOR_FLAG_PROFILE) {
    for (int i = 0; i < ARBOR_NUM_STAGES; ++i)
      for (int r = 0; r < kStageRing; ++r)
        for (int j = 0; j < 2; ++j)
          if (cudaEventCreate(&c->st_ev[i][r][j]) != cudaSuccess) return bail(ARBOR_ERR_CUDA);
    c->st_created = true;
  }
  // pinned host stash [2][L][H][max_tokens][D]
  const size_t stash_bytes = 2ull * c->L * c->H * static_cast<size_t>(c->max_tokens) * c->D * c->esize;
  if (k.host_stash) {
    if (k.host_stash_bytes < stash_bytes) { c->err = "host_stash too small"; return bail(ARBOR_ERR_INVALID_ARG); }
    c->stash_host = k.host_stash;
  } else {
    if (cudaHostAlloc(&c->stash_host, stash_bytes, cudaHostAllocMapped | cudaHostAllocPortable) != cudaSuccess)
      return bail(ARBOR_ERR_IO);
    c->own_stash = true;
  }
  if (cudaHostGetDevicePointer(&c->stash_dev, c->stash_host, 0) != cudaSuccess) return bail(ARBOR_ERR_IO);
  // NCCL communicator for the mass all-reduce (a10)
  if ((k.world_size > 1 || coll) && !ext_reduce) {
    if (!g_nccl.load()) return bail(ARBOR_ERR_NCCL);
    ncclUniqueId id;
    std::memcpy(&id, k.nccl_unique_id, sizeof(id));
    ncclComm_t comm = nullptr;
    if (g_nccl.commInitRank(&comm, k.world_size, id, k.rank) != ncclSuccess) return bail(ARBOR_ERR_NCCL);
    c->nccl_comm = comm;
  }
  attn_tc_init(c);   // tcgen05 attention when the shape allows it (else the CUDA-core kernel)
  if (cudaStreamSynchronize(c->ms) != cudaSuccess) return bail(ARBOR_ERR_CUDA);
  *out = c;
  return ARBOR_OK;
}

void arbor_destroy(arbor_ctx *c) {
  if (c && c->capturing) {   // abandon an unfinished capture
    cudaGraph_t g = nullptr;
    cudaStreamEndCapture(c->ms, &g);
    if (g) cudaGraphDestroy(g);
    c->ms = c->saved_ms;
    c->capturing = false;
    for (void *b : c->cap_bufs) cudaFreeHost(b);
    c->cap_bufs.clear();
  }
  if (c && c->cap_stream) {
    cudaStreamDestroy(c->cap_stream);
    c->cap_stream = nullptr;
  }
  if (!c) return;
  if (c->ms) cudaStreamSynchronize(c->ms);
  if (c->ss) cudaStreamSynchronize(c->ss);
  if (c->nccl_comm && g_nccl.commDestroy) g_nccl.commDestroy(static_cast<ncclComm_t>(c->nccl_comm));
  DevState &d = c->d;
  if (c->unc_part) cudaFree(c->unc_part);
  if (c->unc_ticket) cudaFree(c->unc_ticket);
  void *ptrs[] = {d.n, d.kcur, d.npages, d.soff, d.ptab, d.free_stack, d.span, d.mass2, d.mclose, d.nq,
                  d.a, d.s, d.ctrl, d.parent, d.onpath, d.pinned, d.depth, d.delta, d.Ed, d.ED,
                  d.work, d.rehyd_nodes, d.rehyd_flag, d.seg,
                  d.partials, d.lse_scratch, d.out_scratch, d.zbuf, d.mass_part, d.mass_scratch,
                  d.mass_acc, d.ticket, d.row_done, d.ahat};
  for (void *p : ptrs) if (p) cudaFree(p);
  for (auto &sn : c->snap) {
    if (!sn.valid) continue;
    void *sp[] = {sn.n, sn.kcur, sn.npages, sn.soff, sn.ptab, sn.free_stack, sn.mclose, sn.nq_dev, sn.s, sn.ctrl,
                  sn.mass_part};
    for (void *p : sp) if (p) cudaFree(p);
  }
  for (int i = 0; i < kRingSlots; ++i) {
    if (c->ring[i]) cudaFreeHost(c->ring[i]);
    if (c->ring_ev[i]) cudaEventDestroy(c->ring_ev[i]);
  }
  if (c->ev_main_to_side) cudaEventDestroy(c->ev_main_to_side);
  if (c->ev_side_done) cudaEventDestroy(c->ev_side_done);
  if (c->ev_rehyd_done) cudaEventDestroy(c->ev_rehyd_done);
  if (c->ev_stash_done) cudaEventDestroy(c->ev_stash_done);
  if (c->st_created)
    for (int i = 0; i < ARBOR_NUM_STAGES; ++i)
      for (int r = 0; r < kStageRing; ++r)
        for (int j = 0; j < 2; ++j) if (c->st_ev[i][r][j]) cudaEventDestroy(c->st_ev[i][r][j]);
  if (c->own_stash && c->stash_host) cudaFreeHost(c->stash_host);
  if (c->rehyd_scratch) cudaFree(c->rehyd_scratch);
  if (c->own_ms) cudaStreamDestroy(c->ms);
  if (c->own_ss) cudaStreamDestroy(c->ss);
  delete c;
}

// ---------------------------------------------------------------- node plumbing
arbor_status arbor_open_node(arbor_ctx *c, int32_t node, int64_t span_start) {
  if (!c) return ARBOR_ERR_INVALID_ARG;
  if (node != c->num_known) return fail(c, ARBOR_ERR_INVALID_ARG, "node ids are dense: expected " + std::to_string(c->num_known));
  if (node >= c->max_nodes) return fail(c, ARBOR_ERR_INVALID_ARG, "max_nodes exceeded");
  if (span_start < 0 || span_start >= c->max_tokens) return fail(c, ARBOR_ERR_INVALID_ARG, "span_start out of range");
  // token spans of all nodes are disjoint ranges of the absolute position stream (the
  // accumulated-attention array A is dense by absolute position)
  for (int j = 0; j < c->num_known; ++j)
    if (span_start >= c->h_span[j] && span_start < c->h_span[j] + c->h_n[j])
      return fail(c, ARBOR_ERR_INVALID_ARG, "span_start lies inside node " + std::to_string(j) + "'s span");
  init_node_kernel<<<1, 1, 0, c->ms>>>(node, span_start, c->d.n, c->d.kcur, c->d.npages, c->d.soff, c->d.span,
                                       c->d.mclose, c->d.s, c->d.a);
  ARBOR_LAUNCHED(c);
  CK_LAUNCH();
  ++c->epoch;
  c->h_n.push_back(0);
  c->h_open.push_back(1);
  c->h_span.push_back(span_start);
  c->h_nq.push_back(0);
  ++c->num_known;
  c->tree_valid = false;
  return ARBOR_OK;
}

arbor_status arbor_append_kv(arbor_ctx *c, int32_t node, const void *k, const void *v, int32_t ntok) {
  if (!c) return ARBOR_ERR_INVALID_ARG;
  if (node < 0 || node >= c->num_known) return fail(c, ARBOR_ERR_INVALID_ARG, "unknown node");
  if (!c->h_open[node]) return fail(c, ARBOR_ERR_STATE, "append to a closed node");
  if (ntok < 1 || !k || !v) return fail(c, ARBOR_ERR_INVALID_ARG, "ntok >= 1 and K/V pointers required");
  const int64_t new_n = static_cast<int64_t>(c->h_n[node]) + ntok;
  if (new_n > c->cfg.max_node_tokens) return fail(c, ARBOR_ERR_INVALID_ARG, "node exceeds max_node_tokens");
  if (c->h_span[node] + new_n > c->max_tokens) return fail(c, ARBOR_ERR_INVALID_ARG, "position stream exceeds max_tokens");
  {
    const int64_t lo = c->h_span[node] + c->h_n[node], hi = c->h_span[node] + new_n;
    for (int j = 0; j < c->num_known; ++j)
      if (j != node && c->h_span[j] < hi && c->h_span[j] + std::max<int64_t>(c->h_n[j], 1) > lo)
        return fail(c, ARBOR_ERR_INVALID_ARG, "append would overlap node " + std::to_string(j) + "'s span");
  }
  launch_append(c, node, k, v, c->h_n[node], ntok);
  CK_LAUNCH();
  c->h_n[node] = static_cast<int32_t>(new_n);
  c->tree_valid = false;
  ++c->epoch;
  return ARBOR_OK;
}

arbor_status arbor_close_node(arbor_ctx *c, int32_t node) {
  if (!c) return ARBOR_ERR_INVALID_ARG;
  if (node < 0 || node >= c->num_known) return fail(c, ARBOR_ERR_INVALID_ARG, "unknown node");
  if (!c->h_open[node]) return fail(c, ARBOR_ERR_STATE, "closing a node that is not open");
  if (c->h_n[node] < 1) return fail(c, ARBOR_ERR_INVALID_ARG, "closing an empty node");
  // Mclose_i: this rank's partial mass of the node at close (Q5)
  TRY(ring_upload(c, c->d.rehyd_nodes + c->max_nodes, &node, sizeof(int32_t)));
  launch_node_mass(c, c->d.rehyd_nodes + c->max_nodes, 1, c->d.mclose, 1);
  CK_LAUNCH();
  // the node's cached partial mass starts at its close-time value
  CK(cudaMemcpyAsync(c->d.mass_part + node, c->d.mclose + node, sizeof(int64_t),
                     cudaMemcpyDeviceToDevice, c->ms));
  ++c->epoch;
  // write-through stash on the side stream (a7), after the node's last append
  CK(cudaEventRecord(c->ev_main_to_side, c->ms));
  CK(cudaStreamWaitEvent(c->ss, c->ev_main_to_side, 0));
  launch_stash(c, node, c->h_n[node], c->h_span[node]);
  CK_LAUNCH();
  CK(cudaEventRecord(c->ev_side_done, c->ss));
  CK(cudaEventRecord(c->ev_stash_done, c->ss));
  c->stash_pending = true;
  c->side_pending = true;
  c->h_open[node] = 0;
  c->h_nq[node] = 0;
  c->tree_valid = false;
  return ARBOR_OK;
}

// ---------------------------------------------------------------- hot path
// Per score call: Nq_i += 1 for every closed i on Path(ℓ_b) (one query per active leaf and
// step); the nodes whose partial masses are (re)computed — the visible closed nodes, or all
// closed nodes when the cache is invalid (A changes only at visible tokens).
static void score_bookkeeping(arbor_ctx *c, const arbor_tree *tree, const HostPlan &hp,
                              std::vector<int32_t> &mass_nodes) {
  const int N = tree->num_nodes, nA = tree->num_active;
  std::vector<uint8_t> vis(N, 0);
  for (int b = 0; b < nA; ++b)
    for (int x : hp.paths[b]) {
      vis[x] = 1;
      if (!c->h_open[x]) c->h_nq[x] += 1;
    }
  for (int i = 0; i < N; ++i)
    if (!c->h_open[i] && (vis[i] || !c->mass_valid)) mass_nodes.push_back(i);
}

// split of each row's score pass over CTAs (score.cu score_row: part p takes the plan's
// chunks p, p + parts, …; the row's last part computes its node masses): about 16 chunks per
// part, ≤ 8 parts (a power of two), and never more CTAs than one resident wave (2 per SM) —
// a second wave costs the whole per-CTA latency chain again (decode_post phase trace, C3:
// 2 parts 83 µs vs 1 part 67 µs)
static int score_parts(const arbor_ctx *c, size_t chunks) {
  const int want = std::max(1, std::min(8, static_cast<int>(chunks) / 16));
  int p = 1;
  while (p * 2 <= want) p *= 2;
  while (p > 1 && c->L * c->H * p > kPostCtasPerSm * c->num_sms) p /= 2;
  return p;
}

// the fused single-rank finisher (MSVE inside the score / decode_post kernel) applies
static bool single_rank(const arbor_ctx *c) {
  return c->cfg.world_size == 1 && !(c->cfg.flags & ARBOR_FLAG_COLLECTIVE);
}

// a10 + MSVE on several ranks: the all-reduce sits between the partial masses and the score
// (ARBOR_FLAG_EXTERNAL_REDUCE: the caller's collective, then arbor_score_finish)
static arbor_status score_allreduce(arbor_ctx *c, int N, float *s_out) {
  if (c->cfg.flags & ARBOR_FLAG_EXTERNAL_REDUCE) {
    c->reduce_pending_n = N;
    return ARBOR_OK;
  }
  stage_begin(c, ARBOR_ST_ALLREDUCE, c->ms);
  if (g_nccl.allReduce(c->d.mass2, c->d.mass2, 2 * static_cast<size_t>(N), ncclInt64, ncclSum,
                       static_cast<ncclComm_t>(c->nccl_comm), c->ms) != ncclSuccess)
    return fail(c, ARBOR_ERR_NCCL, "ncclAllReduce failed");
  stage_end(c, ARBOR_ST_ALLREDUCE, c->ms);
  launch_msve(c, N, s_out);
  CK_LAUNCH();
  return ARBOR_OK;
}

arbor_status arbor_score(arbor_ctx *c, const arbor_tree *tree, const void *q, const float *lse,
                         float *s_out) {
  if (!c) return ARBOR_ERR_INVALID_ARG;
  TRY(check_tree(c, tree));
  if (!q) return fail(c, ARBOR_ERR_INVALID_ARG, "q is NULL");
  const int N = tree->num_nodes, nA = tree->num_active;
  TRY(upload_tree(c, tree));
  HostPlan hp;
  build_plan(tree, c->h_n, hp, c->tc_ok);
  std::vector<int32_t> mass_nodes;
  score_bookkeeping(c, tree, hp, mass_nodes);
  PlanView pv{};
  const int32_t *d_mass_nodes = nullptr;
  TRY(upload_plan(c, hp, nA, true, &mass_nodes, pv, &d_mass_nodes));
  // a9's logits are reused when this call follows a full-range arbor_tree_decode_attn with
  // the same q and lse buffers and nothing changed the KV in between (fused a2)
  const bool fused = lse && q == c->lg_q && lse == c->lg_lse && c->lg_epoch == c->epoch &&
                     c->lg_tree == c->tree_version;
  const float *lse_use = lse;
  if (!fused) {
    const size_t qn = static_cast<size_t>(nA) * c->L * c->Hq;
    if (qn > c->scratch_q) {
      if (c->d.lse_scratch) cudaFree(c->d.lse_scratch);
      if (c->d.out_scratch) cudaFree(c->d.out_scratch);
      CK(cudaMalloc(&c->d.lse_scratch, qn * sizeof(float)));
      CK(cudaMalloc(&c->d.out_scratch, qn * c->D * c->esize));
      c->scratch_q = qn;
    }
    TRY(run_attention(c, hp, pv, 0, c->L, q, c->d.out_scratch, c->d.lse_scratch));
    if (!lse) lse_use = c->d.lse_scratch;
  }
  // a2 + a3 in one launch (score.cu): score pass, partial masses, Mass/Mclose → mass2, and —
  // single rank — the MSVE score; with several ranks the all-reduce sits before the MSVE
  const bool single = single_rank(c);
  launch_score_fused(c, pv, lse_use, d_mass_nodes, static_cast<int>(mass_nodes.size()), N, single,
                     s_out, score_parts(c, hp.ch_node.size()));
  CK_LAUNCH();
  c->lg_epoch = -1;   // A changed: the logits must not be applied twice
  c->mass_valid = true;
  if (!single) TRY(score_allreduce(c, N, s_out));
  return ARBOR_OK;
}

// f2: a9 + a2 + a3 as two launches — the attention kernel (partials + logits), then one
// kernel that merges the partials into out / LSE and, with the merged LSE still on chip,
// applies the score pass, the partial masses and (single rank) the MSVE score.  Same
// results as arbor_tree_decode_attn (full layer range) followed by arbor_score.
arbor_status arbor_decode_step(arbor_ctx *c, const arbor_tree *tree, const void *q, void *out,
                               float *lse_out, float *s_out) {
  if (!c) return ARBOR_ERR_INVALID_ARG;
  static const bool htrace = getenv("ARBOR_HOST_TRACE") != nullptr;   // diagnostics
  using clk = std::chrono::steady_clock;
  clk::time_point ht[8];
  int hn = 0;
  auto mark = [&]() {
    if (htrace) {
      ht[hn++] = clk::now();
      static const bool hverbose = getenv("ARBOR_HOST_TRACE_VERBOSE") != nullptr;
      if (hverbose) { fprintf(stderr, "[arbor host] mark %d\n", hn); fflush(stderr); }
    }
  };
  mark();
  TRY(check_tree(c, tree));
  mark();
  if (!q || !out) return fail(c, ARBOR_ERR_INVALID_ARG, "q / out is NULL");
  const int N = tree->num_nodes, nA = tree->num_active;
  if (!decode_post_fits(c, nA)) {   // more (leaf, q-head) pairs than the merge keeps on chip
    TRY(arbor_tree_decode_attn(c, tree, 0, c->L, q, out, lse_out));
    if (lse_out) return arbor_score(c, tree, q, lse_out, s_out);
    return arbor_score(c, tree, q, nullptr, s_out);
  }
  mark();
  HostPlan hp;
  build_plan(tree, c->h_n, hp, c->tc_ok);
  std::vector<int32_t> mass_nodes;
  score_bookkeeping(c, tree, hp, mass_nodes);
  mark();
  PlanView pv{};
  const int32_t *d_mass_nodes = nullptr;
  // the tree mirror rides in the plan's copy (upload_plan)
  TRY(upload_plan(c, hp, nA, true, &mass_nodes, pv, &d_mass_nodes, tree));
  TRY(ensure_partials(c, hp.pair_b.size(), c->L));
  mark();
  wait_rehydrated(c);
  launch_attn_partial(c, pv, q, 0, c->L, hp.max_cnt, out, lse_out);
  CK_LAUNCH();
  mark();
  const bool single = single_rank(c);
  int parts = score_parts(c, hp.ch_node.size());
  static const int parts_env = getenv("ARBOR_POST_PARTS") ? atoi(getenv("ARBOR_POST_PARTS")) : 0;
  if (parts_env > 0) parts = parts_env;   // diagnostics
  launch_decode_post(c, pv, out, lse_out, d_mass_nodes, static_cast<int>(mass_nodes.size()), N,
                     single, s_out, parts);
  CK_LAUNCH();
  mark();
  if (htrace) {
    fprintf(stderr, "[arbor host] decode_step us: check %.1f upload_tree %.1f plan %.1f upload_plan %.1f attn_launch %.1f post_launch %.1f\n",
            std::chrono::duration<double, std::micro>(ht[1] - ht[0]).count(),
            std::chrono::duration<double, std::micro>(ht[2] - ht[1]).count(),
            std::chrono::duration<double, std::micro>(ht[3] - ht[2]).count(),
            std::chrono::duration<double, std::micro>(ht[4] - ht[3]).count(),
            std::chrono::duration<double, std::micro>(ht[5] - ht[4]).count(),
            std::chrono::duration<double, std::micro>(ht[6] - ht[5]).count());
  }
  c->lg_epoch = -1;
  c->mass_valid = true;
  if (!single) TRY(score_allreduce(c, N, s_out));
  return ARBOR_OK;
}

static arbor_status allocate_impl(arbor_ctx *c, const arbor_tree *tree, const float *s,
                                  int64_t budget, int32_t *k_out, int64_t *min_feasible_out,
                                  int mode, int only_node, bool gated = false) {
  std::vector<int32_t> depth;
  TRY(check_tree(c, tree, &depth));
  if (!k_out) return fail(c, ARBOR_ERR_INVALID_ARG, "k_out is NULL");
  if (budget < 0) return fail(c, ARBOR_ERR_INVALID_ARG, "negative budget");
  if (mode == ARBOR_ALLOC_STREAM && tree->num_active != 1)
    return fail(c, ARBOR_ERR_INVALID_ARG, "alloc_mode STREAM flattens one active path");
  // weights must stay ≤ 2^16 (Q29): bound e^{−λ_d d} e^{−λ_Δ Δ} over the tree's depths
  int maxd = 0;
  for (int x : depth) maxd = std::max(maxd, x);
  double bd = 0, bD = 0;
  for (int x = 0; x <= maxd; ++x) bd = std::max(bd, std::exp(-c->prm.lambda_d * x));
  for (int x = 0; x <= 2 * maxd; ++x) bD = std::max(bD, std::exp(-c->prm.lambda_delta * x));
  if (!(bd * bD <= 65536.0)) return fail(c, ARBOR_ERR_INVALID_ARG, "lambda_d / lambda_delta make weights exceed 2^16");
  arbor_params pm = c->prm;
  pm.alloc_mode = mode;
  const int64_t mf = min_feasible(&pm, tree);
  if (mode != ARBOR_ALLOC_STATIC && budget < mf) {
    if (min_feasible_out) *min_feasible_out = mf;
    return fail(c, ARBOR_ERR_INFEASIBLE_BUDGET, "budget " + std::to_string(budget) +
                                                    " < minimum feasible " + std::to_string(mf));
  }
  TRY(upload_tree(c, tree));
  launch_allocate(c, tree->num_nodes, tree->num_active, s ? s : c->d.s, budget, k_out, mode,
                  only_node, gated);
  CK_LAUNCH();
  c->geom_version = c->tree_version;   // the allocate kernel wrote depth, Δ, Path*, pinned
  return ARBOR_OK;
}

arbor_status arbor_allocate(arbor_ctx *c, const arbor_tree *tree, const float *s, int64_t budget,
                            int32_t *k_out, int64_t *min_feasible_out) {
  if (!c) return ARBOR_ERR_INVALID_ARG;
  return allocate_impl(c, tree, s, budget, k_out, min_feasible_out, c->prm.alloc_mode, -1);
}

static arbor_status evict_impl(arbor_ctx *c, const arbor_tree *tree, const int32_t *k_target,
                               int64_t *evicted_tokens_out, bool gated);

arbor_status arbor_evict(arbor_ctx *c, const arbor_tree *tree, const int32_t *k_target,
                         int64_t *evicted_tokens_out) {
  return evict_impl(c, tree, k_target, evicted_tokens_out, false);
}

static arbor_status evict_impl(arbor_ctx *c, const arbor_tree *tree, const int32_t *k_target,
                               int64_t *evicted_tokens_out, bool gated) {
  if (!c) return ARBOR_ERR_INVALID_ARG;
  TRY(check_tree(c, tree));
  if (!k_target) return fail(c, ARBOR_ERR_INVALID_ARG, "k_target is NULL");
  TRY(upload_tree(c, tree));
  const auto pin = host_pinned(tree, &c->prm);
  int max_n = 0;
  for (int i = 0; i < tree->num_nodes; ++i)
    if (!pin[i]) max_n = std::max(max_n, c->h_n[i]);
  // pending stash copies read pages this call may free; a pending rehydration copy writes
  // the pages of its nodes — only a wait if one of them is not pinned here (the usual
  // Transition, Alg. 2, rehydrates Path* and then evicts off-path nodes: they overlap)
  wait_stash(c);
  if (c->rehyd_pending) {
    for (int x : c->rehyd_list)
      if (x >= tree->num_nodes || !pin[x]) { wait_rehydrated(c); break; }
  }
  ++c->epoch;
  if (c->geom_version != c->tree_version) {   // pinned set of this tree not on the device yet
    launch_geometry(c, tree->num_nodes, tree->num_active);
    CK_LAUNCH();
    c->geom_version = c->tree_version;
  }
  if (c->prm.select_shared) {   // one ranking per block on the slice-summed Â
    launch_ahat(c);
    CK_LAUNCH();
  }
  launch_evict(c, tree->num_nodes, k_target, max_n, gated);
  CK_LAUNCH();
  if (evicted_tokens_out) {
    CK(cudaStreamSynchronize(c->ms));
    long long ev = 0;
    CK(cudaMemcpy(&ev, &c->d.ctrl->evicted, sizeof(ev), cudaMemcpyDeviceToHost));
    *evicted_tokens_out = ev;
    TRY(latched(c));
  }
  return ARBOR_OK;
}

static arbor_status rehydrate_impl(arbor_ctx *c, const arbor_tree *tree, const int32_t *nodes,
                                   int32_t count, int keep_floor);

arbor_status arbor_rehydrate(arbor_ctx *c, const arbor_tree *tree, const int32_t *nodes, int32_t count) {
  return rehydrate_impl(c, tree, nodes, count, 0);
}

static arbor_status rehydrate_impl(arbor_ctx *c, const arbor_tree *tree, const int32_t *nodes,
                                   int32_t count, int keep_floor) {
  if (!c) return ARBOR_ERR_INVALID_ARG;
  TRY(check_tree(c, tree));
  if (count < 0 || (count > 0 && !nodes)) return fail(c, ARBOR_ERR_INVALID_ARG, "bad node list");
  std::vector<int32_t> list(nodes, nodes + count);
  for (int x : list) {
    if (x < 0 || x >= c->num_known) return fail(c, ARBOR_ERR_INVALID_ARG, "unknown node in list");
    if (c->h_open[x]) return fail(c, ARBOR_ERR_STATE, "rehydrating an open node");
  }
  std::sort(list.begin(), list.end());
  list.erase(std::unique(list.begin(), list.end()), list.end());
  if (list.empty() || c->prm.no_rehydrate) return ARBOR_OK;   // f4: irreversible eviction
  int max_n = 0;
  for (int x : list) max_n = std::max(max_n, c->h_n[x]);
  TRY(upload_tree(c, tree));
  TRY(ring_upload(c, c->d.rehyd_nodes, list.data(), list.size() * sizeof(int32_t)));
  // no main-stream wait: the copy follows any pending stash on the side stream (in order),
  // and the plan only pops free pages
  ++c->epoch;
  stage_begin(c, ARBOR_ST_REHYDRATE, c->ms);
  launch_rehydrate_plan(c, static_cast<int>(list.size()), keep_floor);
  CK_LAUNCH();
  CK(cudaEventRecord(c->ev_main_to_side, c->ms));
  CK(cudaStreamWaitEvent(c->ss, c->ev_main_to_side, 0));
  launch_rehydrate_copy(c, static_cast<int>(list.size()), max_n);
  CK_LAUNCH();
  CK(cudaEventRecord(c->ev_side_done, c->ss));
  CK(cudaEventRecord(c->ev_rehyd_done, c->ss));
  c->side_pending = true;
  // no wait here: the next attention launch waits for ev_rehyd_done ("before the next
  // decoding step"), and arbor_evict for the whole side stream, so host work and
  // allocation between the two overlap the PCIe copy
  if (!c->rehyd_pending) c->rehyd_list.clear();
  c->rehyd_list.insert(c->rehyd_list.end(), list.begin(), list.end());
  c->rehyd_pending = true;
  stage_end(c, ARBOR_ST_REHYDRATE, c->ss);
  return ARBOR_OK;
}

// ---------------------------------------------------------------- f1: event-driven controller
arbor_status arbor_policy_event(arbor_ctx *c, const arbor_tree *tree, int32_t kind, int32_t node,
                                int64_t budget, int32_t *k_out, int64_t *min_feasible_out) {
  if (!c) return ARBOR_ERR_INVALID_ARG;
  TRY(check_tree(c, tree));
  if (!k_out) return fail(c, ARBOR_ERR_INVALID_ARG, "k_out is NULL");
  switch (kind) {
    case ARBOR_PUE_BOUNDARY: {
      // Alg. 2 l.3-4: ScoreAllocEvict(i) — Eqs. 2-3 for block i only
      if (node < 0 || node >= tree->num_nodes) return fail(c, ARBOR_ERR_INVALID_ARG, "unknown node");
      if (tree->is_open[node] || (node < c->num_known && c->h_open[node]))
        return fail(c, ARBOR_ERR_STATE, "boundary of an open block");
      TRY(allocate_impl(c, tree, nullptr, budget, k_out, min_feasible_out, ARBOR_ALLOC_STATIC, node));
      return arbor_evict(c, tree, k_out, nullptr);
    }
    case ARBOR_PUE_TRANSITION: {
      // Alg. 2 l.5-21: Path* ← RootToLeaf(ℓ*); rehydrate its evicted blocks; Eqs. 2-3 for the
      // off-path blocks, evicting where k drops (arbor_evict applies min(k_cur, k_new))
      std::vector<uint8_t> on(tree->num_nodes, 0);
      std::vector<int32_t> path;
      for (int b = 0; b < tree->num_active; ++b)
        for (int x = tree->active[b]; x >= 0 && !on[x]; x = tree->parent[x]) on[x] = 1;
      for (int x = 0; x < tree->num_nodes; ++x)
        if (on[x] && !tree->is_open[x]) path.push_back(x);
      // Alg. 2 l.8-14; under k_protect only blocks below their floor min(n, k_protect)
      TRY(rehydrate_impl(c, tree, path.data(), static_cast<int32_t>(path.size()), c->prm.k_protect));
      TRY(allocate_impl(c, tree, nullptr, budget, k_out, min_feasible_out, ARBOR_ALLOC_STATIC, -1));
      return arbor_evict(c, tree, k_out, nullptr);
    }
    case ARBOR_PUE_PRESSURE: {
      // Alg. 2 l.22-30: reallocate the off-path blocks to the budget, then evict
      const int mode = c->prm.alloc_mode == ARBOR_ALLOC_WATERFILL ? ARBOR_ALLOC_WATERFILL
                                                                   : ARBOR_ALLOC_STATIC_DRAIN;
      TRY(allocate_impl(c, tree, nullptr, budget, k_out, min_feasible_out, mode, -1));
      return arbor_evict(c, tree, k_out, nullptr);
    }
    default:
      return fail(c, ARBOR_ERR_INVALID_ARG, "unknown policy event");
  }
}

arbor_status arbor_boundary_uncertainty(arbor_ctx *c, const void *logits, int32_t dtype,
                                        int32_t batch, int32_t vocab, float *u_out) {
  if (!c) return ARBOR_ERR_INVALID_ARG;
  if (!logits || !u_out) return fail(c, ARBOR_ERR_INVALID_ARG, "logits / u_out is NULL");
  if (batch < 1 || vocab < 2) return fail(c, ARBOR_ERR_INVALID_ARG, "need batch >= 1 and vocab >= 2");
  if (dtype != ARBOR_F32 && dtype != ARBOR_BF16) return fail(c, ARBOR_ERR_INVALID_ARG, "bad dtype");
  const arbor_status s = launch_uncertainty(c, logits, dtype, batch, vocab, u_out);
  if (s != ARBOR_OK) return fail(c, s, "uncertainty launch failed");
  CK_LAUNCH();
  return ARBOR_OK;
}

// f1: Alg. 2 l.31-33 on the device — no host sync per decode step.  The waterline kernel
// compares M = Σ_i k_cur_i with 𝓑 − δ and gates a Pressure (allocation in the bundle's
// Pressure mode + evict) that is enqueued unconditionally behind it; when the gate is 0 the
// allocation writes k = k_cur and the eviction finds nothing to do.  The Pressure runs in the
// same call, so at most one is ever pending.
arbor_status arbor_policy_waterline(arbor_ctx *c, const arbor_tree *tree, int64_t budget,
                                    int64_t delta, int32_t *k_out) {
  if (!c) return ARBOR_ERR_INVALID_ARG;
  TRY(check_tree(c, tree));
  if (!k_out) return fail(c, ARBOR_ERR_INVALID_ARG, "k_out is NULL");
  if (budget < 0 || delta < 0) return fail(c, ARBOR_ERR_INVALID_ARG, "negative budget / delta");
  const int mode = c->prm.alloc_mode == ARBOR_ALLOC_WATERFILL ? ARBOR_ALLOC_WATERFILL
                                                               : ARBOR_ALLOC_STATIC_DRAIN;
  arbor_params pm = c->prm;
  pm.alloc_mode = mode;
  const bool infeasible = budget < min_feasible(&pm, tree);
  TRY(upload_tree(c, tree));
  launch_waterline(c, tree->num_nodes, budget - delta, infeasible);
  CK_LAUNCH();
  if (infeasible) return ARBOR_OK;   // a raised Pressure latches ARBOR_ERR_INFEASIBLE_BUDGET
  TRY(allocate_impl(c, tree, nullptr, budget, k_out, nullptr, mode, -1, true));
  return evict_impl(c, tree, k_out, nullptr, true);
}

arbor_status arbor_pressure_events(arbor_ctx *c, int64_t *count) {
  if (!c || !count) return ARBOR_ERR_INVALID_ARG;
  TRY(sync_all(c));
  long long v = 0;
  CK(cudaMemcpy(&v, &c->d.ctrl->pressure_events, sizeof(v), cudaMemcpyDeviceToHost));
  *count = v;
  return ARBOR_OK;
}

arbor_status arbor_retained_tokens(arbor_ctx *c, int64_t *total) {
  if (!c || !total) return ARBOR_ERR_INVALID_ARG;
  TRY(sync_all(c));
  std::vector<int32_t> kc(std::max(c->num_known, 1));
  if (c->num_known)
    CK(cudaMemcpy(kc.data(), c->d.kcur, c->num_known * sizeof(int32_t), cudaMemcpyDeviceToHost));
  int64_t t = 0;
  for (int i = 0; i < c->num_known; ++i) t += kc[i];
  *total = t;
  return ARBOR_OK;
}

arbor_status arbor_tree_decode_attn(arbor_ctx *c, const arbor_tree *tree, int32_t layer_begin,
                                    int32_t layer_count, const void *q, void *out, float *lse_out) {
  if (!c) return ARBOR_ERR_INVALID_ARG;
  TRY(check_tree(c, tree));
  if (!q || !out) return fail(c, ARBOR_ERR_INVALID_ARG, "q / out is NULL");
  if (layer_begin < 0 || layer_count < 1 || layer_begin + layer_count > c->L)
    return fail(c, ARBOR_ERR_INVALID_ARG, "layer range outside the shard");
  TRY(upload_tree(c, tree));
  HostPlan hp;
  build_plan(tree, c->h_n, hp, c->tc_ok);
  PlanView pv{};
  TRY(upload_plan(c, hp, tree->num_active, false, nullptr, pv, nullptr));
  TRY(run_attention(c, hp, pv, layer_begin, layer_count, q, out, lse_out));
  const bool full = layer_begin == 0 && layer_count == c->L && lse_out;
  c->lg_q = full ? q : nullptr;
  c->lg_lse = full ? lse_out : nullptr;
  c->lg_epoch = full ? c->epoch : -1;
  c->lg_tree = c->tree_version;
  return ARBOR_OK;
}

// ---------------------------------------------------------------- inspection
arbor_status arbor_sync(arbor_ctx *c) {
  if (!c) return ARBOR_ERR_INVALID_ARG;
  return sync_all(c);
}

arbor_status arbor_read_node(arbor_ctx *c, int32_t node, int32_t *k_cur, int32_t *n, int32_t *pages,
                             int32_t *num_pages) {
  if (!c) return ARBOR_ERR_INVALID_ARG;
  if (node < 0 || node >= c->num_known) return fail(c, ARBOR_ERR_INVALID_ARG, "unknown node");
  TRY(sync_all(c));
  int32_t kc = 0, nn = 0, np = 0, so = 0;
  CK(cudaMemcpy(&kc, c->d.kcur + node, 4, cudaMemcpyDeviceToHost));
  CK(cudaMemcpy(&nn, c->d.n + node, 4, cudaMemcpyDeviceToHost));
  CK(cudaMemcpy(&np, c->d.npages + node, 4, cudaMemcpyDeviceToHost));
  CK(cudaMemcpy(&so, c->d.soff + node, 4, cudaMemcpyDeviceToHost));
  const int first = so / c->P;   // pages before it were freed by an eviction (Q23*)
  np -= first;
  if (k_cur) *k_cur = kc;
  if (n) *n = nn;
  if (num_pages) {
    if (pages) {
      if (*num_pages < np) return fail(c, ARBOR_ERR_INVALID_ARG, "pages buffer too small");
      if (np) CK(cudaMemcpy(pages, c->d.ptab + static_cast<int64_t>(node) * c->max_pages_node + first, np * 4, cudaMemcpyDeviceToHost));
    }
    *num_pages = np;
  }
  return ARBOR_OK;
}

arbor_status arbor_read_node_offset(arbor_ctx *c, int32_t node, int32_t *first_slot) {
  if (!c || !first_slot) return ARBOR_ERR_INVALID_ARG;
  if (node < 0 || node >= c->num_known) return fail(c, ARBOR_ERR_INVALID_ARG, "unknown node");
  TRY(sync_all(c));
  int32_t so = 0;
  CK(cudaMemcpy(&so, c->d.soff + node, 4, cudaMemcpyDeviceToHost));
  *first_slot = so % c->P;
  return ARBOR_OK;
}

arbor_status arbor_read_free_list(arbor_ctx *c, int32_t *pages, int32_t *count) {
  if (!c || !count) return ARBOR_ERR_INVALID_ARG;
  TRY(sync_all(c));
  Ctrl h{};
  CK(cudaMemcpy(&h, c->d.ctrl, sizeof(h), cudaMemcpyDeviceToHost));
  if (pages) {
    if (*count < h.free_top) return fail(c, ARBOR_ERR_INVALID_ARG, "buffer too small");
    if (h.free_top) CK(cudaMemcpy(pages, c->d.free_stack, h.free_top * 4, cudaMemcpyDeviceToHost));
  }
  *count = h.free_top;
  return ARBOR_OK;
}

arbor_status arbor_read_scores(arbor_ctx *c, int32_t num_nodes, int64_t *mass, int64_t *mclose,
                               int64_t *nq, float *a, float *s) {
  if (!c || num_nodes < 0 || num_nodes > c->num_known) return ARBOR_ERR_INVALID_ARG;
  TRY(sync_all(c));
  const int N = num_nodes;
  if (mass && N) CK(cudaMemcpy(mass, c->d.mass2, N * 8, cudaMemcpyDeviceToHost));
  if (mclose && N) CK(cudaMemcpy(mclose, c->d.mclose, N * 8, cudaMemcpyDeviceToHost));
  if (nq) for (int i = 0; i < N; ++i) nq[i] = c->h_nq[i];
  if (a && N) CK(cudaMemcpy(a, c->d.a, N * 4, cudaMemcpyDeviceToHost));
  if (s && N) CK(cudaMemcpy(s, c->d.s, N * 4, cudaMemcpyDeviceToHost));
  return ARBOR_OK;
}

arbor_status arbor_rehydrate_in_flight(arbor_ctx *c, int32_t *in_flight) {
  if (!c || !in_flight) return ARBOR_ERR_INVALID_ARG;
  const cudaError_t e = cudaEventQuery(c->ev_rehyd_done);
  if (e != cudaSuccess && e != cudaErrorNotReady) CK(e);
  *in_flight = e == cudaErrorNotReady ? 1 : 0;
  return ARBOR_OK;
}

arbor_status arbor_mass_buffer(arbor_ctx *c, int64_t **dev, int32_t *count) {
  if (!c || !dev || !count) return ARBOR_ERR_INVALID_ARG;
  *dev = c->d.mass2;
  *count = 2 * (c->reduce_pending_n >= 0 ? c->reduce_pending_n : c->num_known);
  return ARBOR_OK;
}

arbor_status arbor_score_finish(arbor_ctx *c, const int64_t *reduced, float *s_out) {
  if (!c) return ARBOR_ERR_INVALID_ARG;
  if (!(c->cfg.flags & ARBOR_FLAG_EXTERNAL_REDUCE) || c->reduce_pending_n < 0)
    return fail(c, ARBOR_ERR_STATE, "arbor_score_finish: no score awaits an external reduction");
  const int N = c->reduce_pending_n;
  if (reduced && reduced != c->d.mass2)
    CK(cudaMemcpyAsync(c->d.mass2, reduced, 2 * static_cast<size_t>(N) * sizeof(int64_t),
                       cudaMemcpyDeviceToDevice, c->ms));
  launch_msve(c, N, s_out);
  CK_LAUNCH();
  c->reduce_pending_n = -1;
  return ARBOR_OK;
}

arbor_status arbor_read_counters(arbor_ctx *c, int64_t *rehydrations, int64_t *pages_in_use) {
  if (!c) return ARBOR_ERR_INVALID_ARG;
  TRY(sync_all(c));
  Ctrl h{};
  CK(cudaMemcpy(&h, c->d.ctrl, sizeof(h), cudaMemcpyDeviceToHost));
  if (rehydrations) *rehydrations = h.rehydrations;
  if (pages_in_use) *pages_in_use = h.pages_in_use;
  return ARBOR_OK;
}

arbor_status arbor_save_state(arbor_ctx *c, int32_t slot) {
  if (!c || slot < 0 || slot >= kStashSlots) return ARBOR_ERR_INVALID_ARG;
  Snapshot &sn = c->snap[slot];
  const size_t MN = c->max_nodes, PT = MN * c->max_pages_node;
  if (!sn.valid) {
    CK(cudaMalloc(&sn.n, MN * 4)); CK(cudaMalloc(&sn.kcur, MN * 4)); CK(cudaMalloc(&sn.npages, MN * 4));
    CK(cudaMalloc(&sn.soff, MN * 4));
    CK(cudaMalloc(&sn.ptab, PT * 4)); CK(cudaMalloc(&sn.free_stack, c->NP * 4));
    CK(cudaMalloc(&sn.mclose, MN * 8)); CK(cudaMalloc(&sn.nq_dev, MN * 8)); CK(cudaMalloc(&sn.s, MN * 4));
    CK(cudaMalloc(&sn.mass_part, MN * 8));
    CK(cudaMalloc(&sn.ctrl, sizeof(Ctrl)));
    sn.valid = true;
  }
  wait_side(c);
  auto cp = [&](void *dst, const void *src, size_t b) {
    return cudaMemcpyAsync(dst, src, b, cudaMemcpyDeviceToDevice, c->ms);
  };
  CK(cp(sn.n, c->d.n, MN * 4)); CK(cp(sn.kcur, c->d.kcur, MN * 4)); CK(cp(sn.npages, c->d.npages, MN * 4));
  CK(cp(sn.soff, c->d.soff, MN * 4));
  CK(cp(sn.ptab, c->d.ptab, PT * 4)); CK(cp(sn.free_stack, c->d.free_stack, c->NP * 4));
  CK(cp(sn.mclose, c->d.mclose, MN * 8)); CK(cp(sn.s, c->d.s, MN * 4)); CK(cp(sn.ctrl, c->d.ctrl, sizeof(Ctrl)));
  CK(cp(sn.mass_part, c->d.mass_part, MN * 8));
  sn.mass_valid = c->mass_valid;
  sn.h_n = c->h_n; sn.h_open = c->h_open; sn.h_span = c->h_span; sn.h_nq = c->h_nq;
  sn.num_known = c->num_known;
  return ARBOR_OK;
}

arbor_status arbor_load_state(arbor_ctx *c, int32_t slot) {
  if (!c || slot < 0 || slot >= kStashSlots || !c->snap[slot].valid) return ARBOR_ERR_INVALID_ARG;
  Snapshot &sn = c->snap[slot];
  const size_t MN = c->max_nodes, PT = MN * c->max_pages_node;
  wait_side(c);
  auto cp = [&](void *dst, const void *src, size_t b) {
    return cudaMemcpyAsync(dst, src, b, cudaMemcpyDeviceToDevice, c->ms);
  };
  CK(cp(c->d.n, sn.n, MN * 4)); CK(cp(c->d.kcur, sn.kcur, MN * 4)); CK(cp(c->d.npages, sn.npages, MN * 4));
  CK(cp(c->d.soff, sn.soff, MN * 4));
  CK(cp(c->d.ptab, sn.ptab, PT * 4)); CK(cp(c->d.free_stack, sn.free_stack, c->NP * 4));
  CK(cp(c->d.mclose, sn.mclose, MN * 8)); CK(cp(c->d.s, sn.s, MN * 4)); CK(cp(c->d.ctrl, sn.ctrl, sizeof(Ctrl)));
  CK(cp(c->d.mass_part, sn.mass_part, MN * 8));
  c->mass_valid = sn.mass_valid;
  ++c->epoch;
  c->h_n = sn.h_n; c->h_open = sn.h_open; c->h_span = sn.h_span; c->h_nq = sn.h_nq;
  c->num_known = sn.num_known;
  c->tree_valid = false;
  return ARBOR_OK;
}

int64_t arbor_launch_count(const arbor_ctx *c) { return c ? c->launches : 0; }
int32_t arbor_attn_tensor_cores(const arbor_ctx *c) { return c ? (c->tc_ok ? 1 : 0) : -1; }
// ---------------------------------------------------------------- CUDA Graph capture
struct ArborGraph {
  cudaGraphExec_t exec = nullptr;
  std::vector<void *> bufs;   // pinned sources of the captured uploads
};

arbor_status arbor_capture_begin(arbor_ctx *c) {
  if (!c) return ARBOR_ERR_INVALID_ARG;
  if (c->capturing) return fail(c, ARBOR_ERR_STATE, "already capturing");
  TRY(sync_all(c));
  if (c->rehyd_pending || c->stash_pending || c->side_pending) {
    c->rehyd_pending = c->stash_pending = c->side_pending = false;   // both streams are idle
    c->rehyd_list.clear();
  }
  if (!c->cap_stream) CK(cudaStreamCreateWithFlags(&c->cap_stream, cudaStreamNonBlocking));
  c->saved_ms = c->ms;
  c->ms = c->cap_stream;
  c->cap_bufs.clear();
  // the captured calls must not rely on device state the host believes current (the tree
  // mirror, the geometry of this tree): a replay may follow any other work
  c->tree_valid = false;
  ++c->tree_version;
  const cudaError_t e = cudaStreamBeginCapture(c->ms, cudaStreamCaptureModeRelaxed);
  if (e != cudaSuccess) {
    c->ms = c->saved_ms;
    return fail(c, ARBOR_ERR_CUDA, std::string("cudaStreamBeginCapture: ") + cudaGetErrorString(e));
  }
  c->capturing = true;
  return ARBOR_OK;
}

arbor_status arbor_capture_end(arbor_ctx *c, void **graph_out) {
  if (!c || !graph_out) return ARBOR_ERR_INVALID_ARG;
  if (!c->capturing) return fail(c, ARBOR_ERR_STATE, "not capturing");
  cudaGraph_t g = nullptr;
  const cudaError_t e = cudaStreamEndCapture(c->ms, &g);
  c->ms = c->saved_ms;
  c->capturing = false;
  // nothing captured has run: the host's view of the device goes back to "unknown"
  c->tree_valid = false;
  ++c->tree_version;
  c->mass_valid = false;
  auto *ag = new ArborGraph();
  ag->bufs.swap(c->cap_bufs);
  cudaError_t e2 = e;
  if (e == cudaSuccess) {
    e2 = cudaGraphInstantiate(&ag->exec, g, 0);
    cudaGraphDestroy(g);
  }
  if (e2 != cudaSuccess) {
    for (void *b : ag->bufs) cudaFreeHost(b);
    delete ag;
    cudaGetLastError();
    return fail(c, ARBOR_ERR_CUDA, std::string("graph capture: ") + cudaGetErrorString(e2));
  }
  *graph_out = ag;
  return ARBOR_OK;
}

arbor_status arbor_graph_launch(arbor_ctx *c, void *graph) {
  if (!c || !graph) return ARBOR_ERR_INVALID_ARG;
  CK(cudaGraphLaunch(static_cast<ArborGraph *>(graph)->exec, c->ms));
  return ARBOR_OK;
}

arbor_status arbor_graph_destroy(void *graph) {
  if (!graph) return ARBOR_ERR_INVALID_ARG;
  auto *ag = static_cast<ArborGraph *>(graph);
  cudaDeviceSynchronize();
  if (ag->exec) cudaGraphExecDestroy(ag->exec);
  for (void *b : ag->bufs) cudaFreeHost(b);
  delete ag;
  return ARBOR_OK;
}

arbor_status arbor_set_profiling(arbor_ctx *c, int32_t on) {
  if (!c) return ARBOR_ERR_INVALID_ARG;
  if (!(c->cfg.flags & ARBOR_FLAG_PROFILE)) return fail(c, ARBOR_ERR_STATE, "context created without ARBOR_FLAG_PROFILE");
  c->profiling = on != 0;
  return ARBOR_OK;
}

#ifdef ARBOR_ALLOC_TRACE
arbor_status arbor_debug_set_alloc_trace(arbor_ctx *c, long long *trace) {
  c->d.alloc_trace = trace;
  return ARBOR_OK;
}
#endif

arbor_status arbor_invalidate_masses(arbor_ctx *c) {
  if (!c) return ARBOR_ERR_INVALID_ARG;
  c->mass_valid = false;
  c->lg_epoch = -1;
  return ARBOR_OK;
}

arbor_status arbor_stage_times(arbor_ctx *c, float *ms) {
  if (!c || !ms) return ARBOR_ERR_INVALID_ARG;
  TRY(sync_all(c));
  for (int i = 0; i < ARBOR_NUM_STAGES; ++i) {
    ms[i] = 0.f;
    const int n = std::min(c->st_count[i], kStageRing);
    if (!c->st_created || n == 0) continue;
    double tot = 0.0;
    int used = 0;
    for (int r = 0; r < n; ++r) {
      float t = 0.f;
      if (cudaEventElapsedTime(&t, c->st_ev[i][r][0], c->st_ev[i][r][1]) == cudaSuccess) {
        tot += t;
        ++used;
      }
    }
    ms[i] = used ? static_cast<float>(tot / used) : 0.f;
  }
  return ARBOR_OK;
}

arbor_status arbor_reset_stage_times(arbor_ctx *c) {
  if (!c) return ARBOR_ERR_INVALID_ARG;
  for (int i = 0; i < ARBOR_NUM_STAGES; ++i) c->st_count[i] = 0;
  return ARBOR_OK;
}

}  // extern "C"
