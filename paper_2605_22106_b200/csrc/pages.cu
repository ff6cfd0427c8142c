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

// Rehydrate plan: nodes ascending; a node with k_cur < n gets its pages and k_cur = n
// (oracle/state.rehydrate, Q23r).  A closed block's kept window ends at slot n
// (end-window compaction, Q23*: soff + k_cur = n), so the evicted positions go to the slots
// 0 … soff − 1 before it: the ⌊soff/P⌋ stale leading list entries get freshly popped pages (list
// order), the first live page's slots below soff are free already; soff ← 0.  A node evicted
// to 0 (no pages) pops ⌈n/P⌉.  flag[i] = old k_cur + 1 for a restored node, 0 otherwise.
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
    const int kc = kcur[node], nn = n[node];
    if (kc >= nn) continue;   // full: no-op, not counted
    if (keep_floor > 0 && kc >= min(nn, keep_floor)) continue;
    if (kc == 0) {
      soff[node] = 0;
      if (!pop_pages(ctrl, free_stack, npages, ptab, MPN, P, node, nn)) continue;
    } else {
      const int lead = soff[node] / P;
      if (soff[node] + kc != nn || lead > ctrl->free_top) {
        ctrl->err |= soff[node] + kc != nn ? DERR_STATE : DERR_OUT_OF_PAGES;
        continue;
      }
      int32_t *pl = ptab + static_cast<int64_t>(node) * MPN;
      for (int e = 0; e < lead; ++e) pl[e] = free_stack[--ctrl->free_top];
      ctrl->pages_in_use += lead;
      soff[node] = 0;
    }
    flag[i] = kc + 1;
    kcur[node] = nn;
    ++done;
  }
  ctrl->rehydrations += done;
  ctrl->rehyd_count = done;
}

// stash → the evicted rows of each restored node (Q23r): work unit = (listed node,
// row), grid-stride over a small persistent grid (PCIe, not the SMs, is the limit).  The
// k_old kept rows sit in slots n − k_old … n − 1; position p must end in slot p.  Pass 1 reads
// their pos tags into a shared-memory bitmap and stages every kept row that changes slot in
// this CTA's scratch (HBM; its reads of the window all precede pass 2); pass 2 writes the
// staged rows to their slots and copies each missing position from the stash.  Only the
// n − k_old evicted rows cross PCIe (a node evicted to 0: all n).
__global__ void rehydrate_copy_kernel(PoolArgs g, const int32_t *ptab, const int32_t *nodes,
                                      const int32_t *flag, const int32_t *n,
                                      const int64_t *span, const char *stash, char *kpool,
                                      char *vpool, int16_t *pos, int count, char *scratch,
                                      int max_n) {
  extern __shared__ __align__(16) uint32_t rsm[];   // bitmap [nw] | kept positions [max_n] int16
  const int rb = g.D * g.esize, cpr = rb / 16;
  const int lgP = 31 - __clz(g.P), Pm = g.P - 1;
  const int64_t plane = static_cast<int64_t>(g.L) * g.H * g.max_tokens * rb;
  const int rows = g.L * g.H;
  char *stage = scratch + static_cast<int64_t>(blockIdx.x) * max_n * 2 * rb;   // [k][K|V]
  for (int u = blockIdx.x; u < count * rows; u += gridDim.x) {
    const int i = u / rows, r = u - i * rows;
    const int fl = flag[i];
    if (!fl) continue;                   // uniform over the CTA
    const int kold = fl - 1;
    const int node = nodes[i];
    const int nn = n[node], w0 = nn - kold;
    const int l = r / g.H, h = r - l * g.H;
    const int32_t *pl = ptab + static_cast<int64_t>(node) * g.MPN;
    const int64_t a0 = span[node];
    const int nw = (nn + 31) >> 5;
    uint32_t *bits = rsm;
    int16_t *kp = reinterpret_cast<int16_t *>(rsm + nw);
    auto row_of = [&](int slot) { return prow(g, l, pl[slot >> lgP], h, slot & Pm); };
    for (int w = threadIdx.x; w < nw; w += blockDim.x) bits[w] = 0u;
    __syncthreads();
    if (kold > 0) {
      for (int j = threadIdx.x; j < kold; j += blockDim.x) {
        const int p = pos[row_of(w0 + j)];
        kp[j] = static_cast<int16_t>(p);
        if (p >= 0 && p < nn) atomicOr(&bits[p >> 5], 1u << (p & 31));
      }
      __syncthreads();
      for (int idx = threadIdx.x; idx < kold * cpr; idx += blockDim.x) {
        const int j = idx / cpr, cc = idx - j * cpr;
        if (kp[j] == w0 + j) continue;   // already in its slot
        const int64_t src = row_of(w0 + j) * rb + cc * 16;
        char *st = stage + static_cast<int64_t>(j) * 2 * rb + cc * 16;
        *reinterpret_cast<uint4 *>(st) = *reinterpret_cast<const uint4 *>(kpool + src);
        *reinterpret_cast<uint4 *>(st + rb) = *reinterpret_cast<const uint4 *>(vpool + src);
      }
      __syncthreads();                   // every window read is done before any slot is written
      for (int idx = threadIdx.x; idx < kold * cpr; idx += blockDim.x) {
        const int j = idx / cpr, cc = idx - j * cpr;
        const int p = kp[j];
        if (p == w0 + j || p < 0 || p >= nn) continue;
        const int64_t dst = row_of(p);
        const char *st = stage + static_cast<int64_t>(j) * 2 * rb + cc * 16;
        *reinterpret_cast<uint4 *>(kpool + dst * rb + cc * 16) = *reinterpret_cast<const uint4 *>(st);
        *reinterpret_cast<uint4 *>(vpool + dst * rb + cc * 16) = *reinterpret_cast<const uint4 *>(st + rb);
        if (cc == 0) pos[dst] = static_cast<int16_t>(p);
      }
    }
    // the missing positions, from the stash over PCIe (16-byte zero-copy reads)
    for (int idx = threadIdx.x; idx < nn * cpr; idx += blockDim.x) {
      const int p = idx / cpr, cc = idx - p * cpr;
      if (bits[p >> 5] & (1u << (p & 31))) continue;
      const int64_t row = row_of(p);
      const int64_t src = ((static_cast<int64_t>(r)) * g.max_tokens + a0 + p) * rb + cc * 16;
      *reinterpret_cast<uint4 *>(kpool + row * rb + cc * 16) = *reinterpret_cast<const uint4 *>(stash + src);
      *reinterpret_cast<uint4 *>(vpool + row * rb + cc * 16) =
          *reinterpret_cast<const uint4 *>(stash + plane + src);
      if (cc == 0) pos[row] = static_cast<int16_t>(p);
    }
    __syncthreads();                     // the next unit reuses the bitmap, list and staging
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
  const size_t need = static_cast<size_t>(kCopyCtas) * max_n * 2 * c->D * c->esize;
  if (need > c->rehyd_scratch_bytes) {   // grown on first use (a synchronising cudaMalloc)
    if (c->rehyd_scratch) cudaFree(c->rehyd_scratch);
    if (cudaMalloc(&c->rehyd_scratch, need) != cudaSuccess) {
      c->rehyd_scratch = nullptr;
      c->rehyd_scratch_bytes = 0;
      return;                            // the caller's launch check reports the error
    }
    c->rehyd_scratch_bytes = need;
  }
  const int nw = (max_n + 31) / 32;
  const size_t smem = static_cast<size_t>(nw) * 4 + ((static_cast<size_t>(max_n) * 2 + 15) & ~size_t(15));
  if (smem > 48 * 1024)
    cudaFuncSetAttribute(rehydrate_copy_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         static_cast<int>(smem));
  rehydrate_copy_kernel<<<kCopyCtas, 256, smem, c->ss>>>(pool_args(c), c->d.ptab, c->d.rehyd_nodes,
                                                      c->d.rehyd_flag, c->d.n, c->d.span,
                                                      static_cast<const char *>(c->stash_dev),
                                                      static_cast<char *>(c->cfg.k_pool),
                                                      static_cast<char *>(c->cfg.v_pool),
                                                      c->cfg.pos_pool, count,
                                                      static_cast<char *>(c->rehyd_scratch), max_n);
  ARBOR_LAUNCHED(c);
}

}  // namespace arbor
