// pages.cu — paged KV plumbing: append (decode writes), write-through stash (§8(a) a7) and
// lazy rehydration (§8(a) a8).
//
// "Eviction removes KV states but never discards the underlying token
// span … When backtracking makes an evicted block i re-enter the active path, we lazily
// restore its full KV state only at that time … This yields the same conditioning state as
// full retention".  The paper re-prefills; this build restores a bit-exact copy from a
// pinned-host stash written when the block closed (Q20).
//
// Page allocator (Q23, §8(c).1 step 8): per-node page lists (one list shared by every
// (layer, head) row, since k is uniform across rows), a LIFO free stack on the device.  All
// pops happen in single-thread planner kernels in a fixed order (node ascending, token
// order), so page ids are deterministic and identical on every rank.
// Stash / rehydrate copies are SM-driven zero-copy transfers between HBM pages and mapped
// pinned host memory (16-byte loads/stores), on the side stream.
#include "common.cuh"

namespace arbor {
namespace {

struct PoolArgs {
  int L, H, P, D, NP, MPN, esize;
  int64_t max_tokens;
};

__device__ __forceinline__ int64_t prow(const PoolArgs &g, int l, int page, int h, int off) {
  return ((static_cast<int64_t>(l) * g.NP + page) * g.H + h) * g.P + off;
}

// pop pages for `node` so that it can hold new_n slots; single thread
__device__ bool pop_pages(Ctrl *ctrl, int32_t *free_stack, int32_t *npages, int32_t *ptab, int MPN,
                          int P, int node, int new_n) {
  const int need = (new_n + P - 1) / P - npages[node];
  if (need <= 0) return true;
  if (need > ctrl->free_top || (new_n + P - 1) / P > MPN) {
    ctrl->err |= DERR_OUT_OF_PAGES;
    return false;
  }
  int32_t *pl = ptab + static_cast<int64_t>(node) * MPN;
  for (int i = 0; i < need; ++i) {
    const int page = free_stack[--ctrl->free_top];
    pl[npages[node]++] = page;
  }
  ctrl->pages_in_use += need;
  return true;
}

__global__ void append_plan_kernel(Ctrl *ctrl, int32_t *free_stack, int32_t *npages, int32_t *ptab,
                                   int32_t *n, int32_t *kcur, int MPN, int P, int node, int ntok,
                                   int32_t *ok) {
  const int new_n = n[node] + ntok;
  const bool good = pop_pages(ctrl, free_stack, npages, ptab, MPN, P, node, new_n);
  *ok = good ? 1 : 0;
  if (good) {
    n[node] = new_n;
    kcur[node] = new_n;
  }
}

// grid (token chunks, rows): copy ntok rows of K/V [L][H][ntok][D] into the node's slots
__global__ void append_copy_kernel(PoolArgs g, const int32_t *ptab, const int32_t *ok, int node,
                                   int n_old, int ntok, const char *k, const char *v, char *kpool,
                                   char *vpool, int16_t *pos) {
  if (!*ok) return;
  const int r = blockIdx.y;
  const int l = r / g.H, h = r - l * g.H;
  const int rb = g.D * g.esize, cpr = rb / 16;
  const int32_t *pl = ptab + static_cast<int64_t>(node) * g.MPN;
  const int t0 = blockIdx.x * 64;
  const int nt = min(64, ntok - t0);
  for (int idx = threadIdx.x; idx < nt * cpr; idx += blockDim.x) {
    const int tt = idx / cpr, cc = idx - tt * cpr;
    const int t = t0 + tt;
    const int slot = n_old + t;
    const int64_t row = prow(g, l, pl[slot / g.P], h, slot % g.P);
    const int64_t src = ((static_cast<int64_t>(r)) * ntok + t) * rb + cc * 16;
    *reinterpret_cast<uint4 *>(kpool + row * rb + cc * 16) = *reinterpret_cast<const uint4 *>(k + src);
    *reinterpret_cast<uint4 *>(vpool + row * rb + cc * 16) = *reinterpret_cast<const uint4 *>(v + src);
    if (cc == 0) pos[row] = static_cast<int16_t>(slot);
  }
}

// PCIe copies (stash, rehydrate) run on the side stream on a small persistent grid: PCIe
// bandwidth (~50 GB/s) needs ~100 KB of reads in flight, not the whole GPU, and a full-GPU
// grid of long-running zero-copy CTAs would starve the main stream's kernels (allocate, evict)
// that run concurrently with a rehydration (Alg. 2 Transition order).
constexpr int kCopyCtas = 32;

// Stash: node slots 0..n-1 (pos = identity at close) → host [2][L][H][max_tokens][D];
// work unit = (row r, token chunk of 64), grid-stride
__global__ void stash_kernel(PoolArgs g, const int32_t *ptab, int node, int n, int64_t span,
                             const char *kpool, const char *vpool, char *stash) {
  const int rb = g.D * g.esize, cpr = rb / 16;
  const int lgP = 31 - __clz(g.P);
  const int32_t *pl = ptab + static_cast<int64_t>(node) * g.MPN;
  const int nch = (n + 63) / 64;
  const int64_t plane = static_cast<int64_t>(g.L) * g.H * g.max_tokens * rb;
  for (int u = blockIdx.x; u < nch * g.L * g.H; u += gridDim.x) {
    const int r = u / nch, t0 = (u - r * nch) * 64;
    const int l = r / g.H, h = r - l * g.H;
    const int nt = min(64, n - t0);
    for (int idx = threadIdx.x; idx < nt * cpr; idx += blockDim.x) {
      const int tt = idx / cpr, cc = idx - tt * cpr;
      const int slot = t0 + tt;
      const int64_t row = prow(g, l, pl[slot >> lgP], h, slot & (g.P - 1));
      const int64_t dst = ((static_cast<int64_t>(r)) * g.max_tokens + span + slot) * rb + cc * 16;
      *reinterpret_cast<uint4 *>(stash + dst) = *reinterpret_cast<const uint4 *>(kpool + row * rb + cc * 16);
      *reinterpret_cast<uint4 *>(stash + plane + dst) =
          *reinterpret_cast<const uint4 *>(vpool + row * rb + cc * 16);
    }
  }
}

// Rehydrate plan: nodes ascending; a node with k_cur < n gets its pages and k_cur = n.
// Its live pages (from the one holding slot soff, Q23*) move to the front of its
// list and soff = 0, then pages are popped up to ⌈n/P⌉ (oracle/state.rehydrate).
// keep_floor > 0 (the controller's Transition under params.k_protect): only nodes
// below min(n, keep_floor) are restored (to the full span).
__global__ void rehydrate_plan_kernel(Ctrl *ctrl, int32_t *free_stack, int32_t *npages,
                                      int32_t *ptab, const int32_t *n, int32_t *kcur,
                                      int32_t *soff, int MPN, int P, const int32_t *nodes,
                                      int count, int32_t *flag, int keep_floor) {
  int done = 0;
  for (int i = 0; i < count; ++i) {
    const int node = nodes[i];
    flag[i] = 0;
    if (kcur[node] >= n[node]) continue;   // full: no-op, not counted
    if (keep_floor > 0 && kcur[node] >= min(n[node], keep_floor)) continue;
    const int first = soff[node] / P;
    if (first > 0) {
      int32_t *pl = ptab + static_cast<int64_t>(node) * MPN;
      for (int i = first; i < npages[node]; ++i) pl[i - first] = pl[i];
      npages[node] -= first;
    }
    soff[node] = 0;
    if (!pop_pages(ctrl, free_stack, npages, ptab, MPN, P, node, n[node])) continue;
    kcur[node] = n[node];
    flag[i] = 1;
    ++done;
  }
  ctrl->rehydrations += done;
  ctrl->rehyd_count = done;
}

// stash → pages, pos = slot; work unit = (listed node i, row r, token chunk of 64), grid-stride
__global__ void rehydrate_copy_kernel(PoolArgs g, const int32_t *ptab, const int32_t *nodes,
                                      const int32_t *flag, const int32_t *n, const int64_t *span,
                                      const char *stash, char *kpool, char *vpool, int16_t *pos,
                                      int count, int nch) {
  const int rb = g.D * g.esize, cpr = rb / 16;
  const int lgP = 31 - __clz(g.P);
  const int64_t plane = static_cast<int64_t>(g.L) * g.H * g.max_tokens * rb;
  const int rows = g.L * g.H;
  for (int u = blockIdx.x; u < count * rows * nch; u += gridDim.x) {
    const int i = u / (rows * nch);
    const int rem = u - i * rows * nch;
    const int r = rem / nch, t0 = (rem - r * nch) * 64;
    if (!flag[i]) continue;
    const int node = nodes[i];
    const int nn = n[node];
    if (t0 >= nn) continue;
    const int nt = min(64, nn - t0);
    const int l = r / g.H, h = r - l * g.H;
    const int32_t *pl = ptab + static_cast<int64_t>(node) * g.MPN;
    const int64_t a0 = span[node];
    for (int idx = threadIdx.x; idx < nt * cpr; idx += blockDim.x) {
      const int tt = idx / cpr, cc = idx - tt * cpr;
      const int slot = t0 + tt;
      const int64_t row = prow(g, l, pl[slot >> lgP], h, slot & (g.P - 1));
      const int64_t src = ((static_cast<int64_t>(r)) * g.max_tokens + a0 + slot) * rb + cc * 16;
      *reinterpret_cast<uint4 *>(kpool + row * rb + cc * 16) = *reinterpret_cast<const uint4 *>(stash + src);
      *reinterpret_cast<uint4 *>(vpool + row * rb + cc * 16) =
          *reinterpret_cast<const uint4 *>(stash + plane + src);
      if (cc == 0) pos[row] = static_cast<int16_t>(slot);
    }
  }
}

PoolArgs pool_args(arbor_ctx *c) {
  return PoolArgs{c->L, c->H, c->P, c->D, c->NP, c->max_pages_node, c->esize, c->max_tokens};
}

}  // namespace

void launch_append(arbor_ctx *c, int node, const void *k, const void *v, int n_old, int ntok) {
  int32_t *ok = c->d.rehyd_flag + c->max_nodes;   // scratch flag slot
  append_plan_kernel<<<1, 1, 0, c->ms>>>(c->d.ctrl, c->d.free_stack, c->d.npages, c->d.ptab,
                                        c->d.n, c->d.kcur, c->max_pages_node, c->P, node, ntok, ok);
  ARBOR_LAUNCHED(c);
  dim3 grid((ntok + 63) / 64, c->L * c->H);
  append_copy_kernel<<<grid, 256, 0, c->ms>>>(pool_args(c), c->d.ptab, ok, node, n_old, ntok,
                                               static_cast<const char *>(k),
                                               static_cast<const char *>(v),
                                               static_cast<char *>(c->cfg.k_pool),
                                               static_cast<char *>(c->cfg.v_pool), c->cfg.pos_pool);
  ARBOR_LAUNCHED(c);
}

void launch_stash(arbor_ctx *c, int node, int n, int64_t span) {
  stage_begin(c, ARBOR_ST_STASH, c->ss);
  stash_kernel<<<kCopyCtas, 256, 0, c->ss>>>(pool_args(c), c->d.ptab, node, n, span,
                                        static_cast<const char *>(c->cfg.k_pool),
                                        static_cast<const char *>(c->cfg.v_pool),
                                        static_cast<char *>(c->stash_dev));
  ARBOR_LAUNCHED(c);
  stage_end(c, ARBOR_ST_STASH, c->ss);
}

void launch_rehydrate_plan(arbor_ctx *c, int count, int keep_floor) {
  rehydrate_plan_kernel<<<1, 1, 0, c->ms>>>(c->d.ctrl, c->d.free_stack, c->d.npages, c->d.ptab,
                                           c->d.n, c->d.kcur, c->d.soff, c->max_pages_node, c->P,
                                           c->d.rehyd_nodes, count, c->d.rehyd_flag, keep_floor);
  ARBOR_LAUNCHED(c);
}

void launch_rehydrate_copy(arbor_ctx *c, int count, int max_n) {
  if (count == 0 || max_n == 0) return;
  rehydrate_copy_kernel<<<kCopyCtas, 256, 0, c->ss>>>(pool_args(c), c->d.ptab, c->d.rehyd_nodes,
                                                      c->d.rehyd_flag, c->d.n, c->d.span,
                                                      static_cast<const char *>(c->stash_dev),
                                                      static_cast<char *>(c->cfg.k_pool),
                                                      static_cast<char *>(c->cfg.v_pool),
                                                      c->cfg.pos_pool, count, (max_n + 63) / 64);
  ARBOR_LAUNCHED(c);
}

}  // namespace arbor
