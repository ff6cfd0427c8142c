// evict.cu — §8(a) a5+a6: token-extractive selection and in-place paged compaction.
//
// PAPER.md §4 Execution and Alg. 1 procedure Evict: keep the block
// tail 𝒯_i (last min(L_tail, n_i) tokens) and the top-m_i heavy hitters by the
// accumulated attention A_i(t), m_i = k_i − |𝒯_i|; if k_i ≤ L_tail keep the
// last k_i; free the KV of everything else.  Alg. 2: evict only
// where the new k is smaller (k_app = min(k_cur, k_target), Q17).  Per (layer, KV head) row
// (Q1); candidates are the currently kept non-tail slots (Q2); order = 64-bit key
// ⟨f32 bits of A, within-node position⟩ descending (Q3).
//
// B200 design:
//  * evict_plan (1 CTA): decides k_app per node, builds the work list of changed non-pinned
//    nodes in ascending id, truncates page lists to ⌈k_app/P⌉ and pushes the freed pages on
//    the LIFO free list in ascending (node, list) order — all on the device, no host sync.
//  * select (persistent grid, one WARP per (node, row) work item, no block barriers):
//    pos tags + A keys of the kept slots, the m-th largest unique 48-bit key ⟨A bits, pos⟩
//    by a warp radix select (8-bit digits, per-warp smem histogram, warp scan) — exact top-m
//    membership in O(c) — then hole-filling: kept rows inside the new prefix [0, k_app)
//    stay, the i-th hole takes the i-th kept row from beyond it (Q23').  Sources
//    and destinations are disjoint, so the (src, dst) row pairs go to a global list.
//  * move (persistent grid): a pure 16-byte-coalesced streaming copy of the listed K, V
//    rows and pos tags — no ordering constraints, full occupancy.
#include <cub/block/block_scan.cuh>

#include "tile.cuh"

namespace arbor {
namespace {

constexpr int kPlanThreads = 1024;

struct PlanArgs {
  int N, P, MPN;
  const int32_t *k_target;
  const uint8_t *pinned;
  int32_t *kcur, *npages, *ptab, *free_stack;
  int32_t *work_node, *work_old, *work_new;
  Ctrl *ctrl;
};

__global__ void __launch_bounds__(kPlanThreads)
evict_plan_kernel(PlanArgs a) {
  // each thread owns a contiguous block of nodes so that prefix sums keep ascending order
  constexpr int kPer = 4;   // N ≤ 4096
  using Scan = cub::BlockScan<int, kPlanThreads>;
  __shared__ typename Scan::TempStorage tmp;
  __shared__ int tot_work, tot_free;
  __shared__ long long tot_ev;
  if (threadIdx.x == 0) { tot_ev = 0; }
  __syncthreads();
  int kapp[kPer], kc[kPer], ev[kPer], fr[kPer], newp[kPer];
  int my_work = 0, my_free = 0;
  long long my_ev = 0;
#pragma unroll
  for (int i = 0; i < kPer; ++i) {
    const int j = threadIdx.x * kPer + i;
    ev[i] = 0; fr[i] = 0; kc[i] = 0; kapp[i] = 0; newp[i] = 0;
    if (j < a.N) {
      kc[i] = a.kcur[j];
      int kt = a.k_target[j];
      kt = kt < 0 ? 0 : kt;
      kapp[i] = kt < kc[i] ? kt : kc[i];
      if (!a.pinned[j] && kapp[i] < kc[i]) {
        ev[i] = 1;
        newp[i] = (kapp[i] + a.P - 1) / a.P;
        fr[i] = a.npages[j] - newp[i];
      }
    }
    my_work += ev[i];
    my_free += fr[i];
    my_ev += ev[i] ? (kc[i] - kapp[i]) : 0;
  }
  int work_off, free_off;
  Scan(tmp).ExclusiveSum(my_work, work_off);
  __syncthreads();
  Scan(tmp).ExclusiveSum(my_free, free_off);
  __syncthreads();
  atomicAdd(reinterpret_cast<unsigned long long *>(&tot_ev), static_cast<unsigned long long>(my_ev));
  if (threadIdx.x == kPlanThreads - 1) {
    tot_work = work_off + my_work;
    tot_free = free_off + my_free;
  }
  const int top = a.ctrl->free_top;
  __syncthreads();
#pragma unroll
  for (int i = 0; i < kPer; ++i) {
    const int j = threadIdx.x * kPer + i;
    if (!ev[i]) continue;
    a.work_node[work_off] = j;
    a.work_old[work_off] = kc[i];
    a.work_new[work_off] = kapp[i];
    ++work_off;
    a.npages[j] = newp[i];
    a.kcur[j] = kapp[i];
  }
  // freed pages → LIFO free stack, (node, list) ascending: all of a node's page ids are loaded
  // before any store (the stores could alias the page table for the compiler, which would
  // otherwise serialise one global load round trip per page)
#pragma unroll
  for (int i = 0; i < kPer; ++i) {
    const int j = threadIdx.x * kPer + i;
    if (!ev[i] || fr[i] == 0) continue;
    const int32_t *__restrict__ pl = a.ptab + static_cast<int64_t>(j) * a.MPN + newp[i];
    int32_t *__restrict__ dst = a.free_stack + top + free_off;
    constexpr int kB = 16;
    for (int t0 = 0; t0 < fr[i]; t0 += kB) {
      int32_t v[kB];
#pragma unroll
      for (int t = 0; t < kB; ++t) v[t] = t0 + t < fr[i] ? __ldg(pl + t0 + t) : 0;
#pragma unroll
      for (int t = 0; t < kB; ++t) if (t0 + t < fr[i]) dst[t0 + t] = v[t];
    }
    free_off += fr[i];
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    a.ctrl->free_top = top + tot_free;
    a.ctrl->work_count = tot_work;
    a.ctrl->move_count = 0;
    a.ctrl->evicted = tot_ev;
    a.ctrl->pages_in_use -= tot_free;
  }
}

struct CompactArgs {
  int R;            // rows = L * H
  int H, P, D, NP, MPN, l_tail;
  int64_t max_tokens;
  const int32_t *work_node, *work_old, *work_new, *n;
  const int64_t *span;
  const float *A;
  const Ctrl *ctrl_ro;
  Ctrl *ctrl;
  const int32_t *ptab;
  void *kpool, *vpool;
  int16_t *pos;
  int2 *moves;      // (src row, dst row) pairs
  int esize;
  int cap;          // max n over evicted nodes (smem capacity, slots)
  int lgP;          // log2(page size)
};

constexpr int kWarps = 8;     // warps per CTA in the select kernel (one warp per work item)
// fused: each warp streams its own item's moves right after selecting it (other warps'
// selection latency hides under those moves); split: select → global list → move_kernel
constexpr bool kFusedCompact = true;
constexpr bool kWarpSpecialised = true;   // select_move_ws_kernel (below) is the default

// Select: one WARP per (node, row) work item.  Keep = the block tail 𝒯 (positions ≥ n − |𝒯|,
// P:177-182) ∪ the top-m non-tail candidates by the 48-bit key ⟨A bits, pos⟩,
// or the last k_app positions when k_app ≤ |𝒯| (Alg. 1).  The m-th largest key is
// found by a warp radix select (8-bit digits, per-warp 256-bin smem histogram, warp scan):
// exact, O(c).  Slot layout (Q23'): kept rows in slots [0, k_app) stay; the i-th
// hole there takes the i-th kept row from slots ≥ k_app — sources and destinations are
// disjoint, so the moves are appended to a global list and executed by move_kernel.
// smem per warp: key[cap] (u64), hole list[cap], mover list[cap] (u16 pairs), pages.
template <bool kFused>
__global__ void __launch_bounds__(kWarps * 32, kFused ? 4 : 5)
select_kernel(CompactArgs a) {
  extern __shared__ __align__(16) unsigned char sm[];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int cap = a.cap;
  const int lgP = a.lgP, Pm = (1 << lgP) - 1;
  const int pcap = (cap >> lgP) + 1;
  unsigned long long *key = reinterpret_cast<unsigned long long *>(sm) + warp * cap;
  int32_t *holes = reinterpret_cast<int32_t *>(reinterpret_cast<unsigned long long *>(sm) +
                                               kWarps * cap) + warp * 2 * cap;
  int32_t *movers = holes + cap;
  int32_t *pgs = reinterpret_cast<int32_t *>(reinterpret_cast<unsigned long long *>(sm) +
                                             kWarps * cap) + kWarps * 2 * cap + warp * pcap;
  __shared__ uint32_t hist_all[kWarps][256];
  uint32_t *hist = hist_all[warp];
  const int items = a.ctrl_ro->work_count * a.R;
  const unsigned lt_mask = (1u << lane) - 1u;
  const int64_t pstride = static_cast<int64_t>(a.H) << lgP;
  constexpr unsigned long long kCand = 1ull << 63;
  for (int it = blockIdx.x * kWarps + warp; it < items; it += gridDim.x * kWarps) {
    const int w = it / a.R, r = it - w * a.R;
    const int l = r / a.H, h = r - l * a.H;
    const int node = a.work_node[w];
    const int kc = a.work_old[w], ka = a.work_new[w];
    const int n = a.n[node];
    const int tl = min(a.l_tail, n);
    const int32_t *pl = a.ptab + static_cast<int64_t>(node) * a.MPN;
    const int64_t base = (static_cast<int64_t>(l) * a.NP * a.H + h) << lgP;
    for (int i = lane; i < ((kc + Pm) >> lgP); i += 32) pgs[i] = pl[i];
    __syncwarp();
    auto row = [&](int slot) -> int64_t {
      return base + static_cast<int64_t>(pgs[slot >> lgP]) * pstride + (slot & Pm);
    };
    const bool ranked = ka > tl;
    const int m = ka - tl;
    const int tail_from = n - (ranked ? tl : ka);   // keep positions ≥ tail_from outright
    // 1. pos tags of every kept slot; keys of the non-tail candidates (bit 63 = candidate)
    const float *Arow = a.A + (static_cast<int64_t>(l) * a.H + h) * a.max_tokens + a.span[node];
    int ncand = 0;
    for (int s0 = 0; s0 < kc; s0 += 32) {
      const int s = s0 + lane;
      unsigned long long kk = 0;
      if (s < kc) {
        const int p = a.pos[row(s)];
        kk = static_cast<unsigned>(p);   // pos in the low bits; no candidate bit
        if (ranked && p < tail_from) {
          const float av = Arow[p];
          if (!(av >= 0.f) || isinf(av)) atomicOr(&a.ctrl->err, DERR_INVARIANT);
          const unsigned bits = (av == 0.f) ? 0u : __float_as_uint(av);   // −0 → +0 (Q3)
          kk = kCand | (static_cast<unsigned long long>(bits) << 16) | static_cast<unsigned>(p);
        }
        key[s] = kk;
      }
      ncand += __popc(__ballot_sync(0xffffffffu, (kk & kCand) != 0));
    }
    __syncwarp();
    // 2. threshold: keep a candidate iff (key & tmask) >= tkey (the top m unique keys)
    unsigned long long tkey = kCand, tmask = kCand;     // m ≥ ncand: all candidates
    if (ranked && m <= 0) {
      tkey = ~0ull; tmask = ~0ull;                      // none survives
    } else if (ranked && m < ncand) {
      unsigned long long prefix = kCand, pmask = kCand;
      int need = m;
      for (int shift = 40; shift >= 0; shift -= 8) {
#pragma unroll
        for (int b = 0; b < 8; ++b) hist[lane * 8 + b] = 0;
        __syncwarp();
        for (int s = lane; s < kc; s += 32) {
          const unsigned long long k = key[s];
          if ((k & pmask) == prefix) atomicAdd(&hist[(k >> shift) & 255u], 1u);
        }
        __syncwarp();
        uint32_t c[8];
        uint32_t loc = 0;
#pragma unroll
        for (int b = 0; b < 8; ++b) { c[b] = hist[255 - lane * 8 - b]; loc += c[b]; }
        uint32_t incl = loc;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
          const uint32_t t = __shfl_up_sync(0xffffffffu, incl, o);
          if (lane >= o) incl += t;
        }
        const uint32_t before = incl - loc;
        const bool mine = before < static_cast<uint32_t>(need) && static_cast<uint32_t>(need) <= incl;
        int dsel = 0;
        uint32_t above = 0, inbin = 0;
        if (mine) {
          uint32_t acc = before;
#pragma unroll
          for (int b = 0; b < 8; ++b) {
            if (inbin == 0 && acc < static_cast<uint32_t>(need) &&
                static_cast<uint32_t>(need) <= acc + c[b]) {
              dsel = 255 - lane * 8 - b;
              above = acc;
              inbin = c[b];
            }
            acc += c[b];
          }
        }
        const int src = __ffs(__ballot_sync(0xffffffffu, mine)) - 1;
        dsel = __shfl_sync(0xffffffffu, dsel, src);
        above = __shfl_sync(0xffffffffu, above, src);
        inbin = __shfl_sync(0xffffffffu, inbin, src);
        need -= static_cast<int>(above);
        prefix |= static_cast<unsigned long long>(dsel) << shift;
        pmask |= 255ull << shift;
        if (static_cast<uint32_t>(need) == inbin) break;   // the whole bin survives
      }
      tkey = prefix;
      tmask = pmask;
    }
    // 3. keep flags → holes (dropped slots < k_app) and movers (kept slots ≥ k_app), ascending
    int nh = 0, nm = 0;
    for (int s0 = 0; s0 < kc; s0 += 32) {
      const int s = s0 + lane;
      int keep = 0;
      if (s < kc) {
        const unsigned long long k = key[s];
        const int p = static_cast<int>(k & 0xffffu);
        keep = (p >= tail_from) || (ranked && (k & kCand) && (k & tmask) >= tkey);
      }
      const int hole = s < ka && !keep;
      const int mover = s >= ka && s < kc && keep;
      const unsigned hb = __ballot_sync(0xffffffffu, hole);
      const unsigned mb = __ballot_sync(0xffffffffu, mover);
      if (hole) holes[nh + __popc(hb & lt_mask)] = s;
      if (mover) movers[nm + __popc(mb & lt_mask)] = s;
      nh += __popc(hb);
      nm += __popc(mb);
    }
    __syncwarp();
    if (nh != nm && lane == 0) atomicOr(&a.ctrl->err, DERR_STATE);
    if (kFused) {
      // 4'. stream this item's moves directly (disjoint sources/destinations: no barriers)
      const int rb = a.D * a.esize, cpr = rb >> 4, rpi = 32 / cpr;
      const int piece = lane % cpr, sub = lane / cpr;
      char *kp8 = static_cast<char *>(a.kpool);
      char *vp8 = static_cast<char *>(a.vpool);
      constexpr int kU = 4;
      for (int c0 = 0; c0 < nm; c0 += rpi * kU) {
        uint4 bk[kU], bv[kU];
        int64_t srow[kU], drow[kU];
#pragma unroll
        for (int u = 0; u < kU; ++u) {
          const int i = c0 + u * rpi + sub;
          srow[u] = -1;
          if (i < nm) {
            srow[u] = row(movers[i]);
            drow[u] = row(holes[i]);
            bk[u] = *reinterpret_cast<const uint4 *>(kp8 + srow[u] * rb + piece * 16);
            bv[u] = *reinterpret_cast<const uint4 *>(vp8 + srow[u] * rb + piece * 16);
          }
        }
#pragma unroll
        for (int u = 0; u < kU; ++u) {
          if (srow[u] >= 0) {
            *reinterpret_cast<uint4 *>(kp8 + drow[u] * rb + piece * 16) = bk[u];
            *reinterpret_cast<uint4 *>(vp8 + drow[u] * rb + piece * 16) = bv[u];
            if (piece == 0) a.pos[drow[u]] = static_cast<int16_t>(key[movers[c0 + u * rpi + sub]] & 0xffffu);
          }
        }
      }
      __syncwarp();
    } else {
      // 4. append the (src, dst) row pairs to the global move list
      int baseidx = 0;
      if (lane == 0 && nm > 0) baseidx = atomicAdd(&a.ctrl->move_count, nm);
      baseidx = __shfl_sync(0xffffffffu, baseidx, 0);
      for (int i = lane; i < nm; i += 32)
        a.moves[baseidx + i] = make_int2(static_cast<int>(row(movers[i])), static_cast<int>(row(holes[i])));
      __syncwarp();
    }
  }
}

// Warp-specialised select + move (default).  A CTA holds kPairs (select warp, move warp)
// pairs.  Select warp p processes the work items it, it + stride, … exactly like select_kernel
// and hands each item's (src row, dst row) list to its move warp through a 2-slot job queue
// in shared memory guarded by mbarriers (full / empty); move warp p streams those rows (K, V:
// 16-byte coalesced, kUw rows in flight per lane group; pos tags) while its select warp
// already ranks the next item.  Selection (latency-bound) and data movement (HBM-bound) thus
// overlap inside every SM.
constexpr int kPairs = 8;
constexpr int kUw = 4;
__global__ void __launch_bounds__(kPairs * 64, 2)
select_move_ws_kernel(CompactArgs a) {
  extern __shared__ __align__(16) unsigned char sm[];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const bool mover = warp >= kPairs;
  const int pid = mover ? warp - kPairs : warp;
  const int cap = a.cap;
  const int jcap = cap / 2 + 1;                    // moves per item ≤ min(k_app, k_cur − k_app)
  const int lgP = a.lgP, Pm = (1 << lgP) - 1;
  const int pcap = (cap >> lgP) + 1;
  // smem: per select warp key[cap] u64, holes/movers[cap] i32 x2, pages[pcap];
  //       per pair jobs[2][jcap] int2 + counts[2]; mbarriers full[pair][2], empty[pair][2]
  unsigned long long *keys = reinterpret_cast<unsigned long long *>(sm);
  int32_t *lists = reinterpret_cast<int32_t *>(keys + kPairs * cap);
  int32_t *pages_all = lists + kPairs * 2 * cap;
  int2 *jobs = reinterpret_cast<int2 *>(pages_all + ((kPairs * pcap + 1) & ~1));
  int32_t *jcount = reinterpret_cast<int32_t *>(jobs + kPairs * 2 * jcap);
  uint64_t *bars = reinterpret_cast<uint64_t *>(jcount + ((kPairs * 2 + 1) & ~1));
  uint64_t *full = bars + pid * 4, *empty = bars + pid * 4 + 2;
  __shared__ uint32_t hist_all[kPairs][256];
  if (threadIdx.x == 0) {
    for (int i = 0; i < kPairs * 2; ++i) {
      mbar_init(&bars[(i >> 1) * 4 + (i & 1)], 1);
      mbar_init(&bars[(i >> 1) * 4 + 2 + (i & 1)], 1);
    }
    mbar_fence_init();
  }
  __syncthreads();
  const int items = a.ctrl_ro->work_count * a.R;
  const int stride = gridDim.x * kPairs;
  int2 *myjobs = jobs + pid * 2 * jcap;
  int32_t *mycount = jcount + pid * 2;
  if (mover) {
    // ------------------------------------------------------------ move warp
    const int rb = a.D * a.esize, cpr = rb >> 4, rpi = 32 / cpr;
    const int piece = lane % cpr, sub = lane / cpr;
    char *kp8 = static_cast<char *>(a.kpool);
    char *vp8 = static_cast<char *>(a.vpool);
    int k = 0;
    for (int it = blockIdx.x * kPairs + pid; it < items; it += stride, ++k) {
      const int sl = k & 1;
      mbar_wait(&full[sl], (k >> 1) & 1);
      const int nm = mycount[sl];
      const int2 *jb = myjobs + sl * jcap;
      for (int c0 = 0; c0 < nm; c0 += rpi * kUw) {
        uint4 bk[kUw], bv[kUw];
        int2 mv[kUw];
        int16_t pt[kUw];
#pragma unroll
        for (int u = 0; u < kUw; ++u) {
          const int i = c0 + u * rpi + sub;
          mv[u] = i < nm ? jb[i] : make_int2(-1, -1);
          if (mv[u].x >= 0) {
            const int64_t off = static_cast<int64_t>(mv[u].x) * rb + piece * 16;
            bk[u] = *reinterpret_cast<const uint4 *>(kp8 + off);
            bv[u] = *reinterpret_cast<const uint4 *>(vp8 + off);
            if (piece == 0) pt[u] = a.pos[mv[u].x];
          }
        }
#pragma unroll
        for (int u = 0; u < kUw; ++u) {
          if (mv[u].x >= 0) {
            const int64_t off = static_cast<int64_t>(mv[u].y) * rb + piece * 16;
            *reinterpret_cast<uint4 *>(kp8 + off) = bk[u];
            *reinterpret_cast<uint4 *>(vp8 + off) = bv[u];
            if (piece == 0) a.pos[mv[u].y] = pt[u];
          }
        }
      }
      __syncwarp();
      if (lane == 0) mbar_arrive(&empty[sl]);
    }
    return;
  }
  // -------------------------------------------------------------- select warp
  unsigned long long *key = keys + pid * cap;
  int32_t *holes = lists + pid * 2 * cap;
  int32_t *movers = holes + cap;
  int32_t *pgs = pages_all + pid * pcap;
  uint32_t *hist = hist_all[pid];
  const unsigned lt_mask = (1u << lane) - 1u;
  const int64_t pstride = static_cast<int64_t>(a.H) << lgP;
  constexpr unsigned long long kCand = 1ull << 63;
  int k = 0;
  for (int it = blockIdx.x * kPairs + pid; it < items; it += stride, ++k) {
    const int w = it / a.R, r = it - w * a.R;
    const int l = r / a.H, h = r - l * a.H;
    const int node = a.work_node[w];
    const int kc = a.work_old[w], ka = a.work_new[w];
    const int n = a.n[node];
    const int tl = min(a.l_tail, n);
    const int32_t *pl = a.ptab + static_cast<int64_t>(node) * a.MPN;
    const int64_t base = (static_cast<int64_t>(l) * a.NP * a.H + h) << lgP;
    for (int i = lane; i < ((kc + Pm) >> lgP); i += 32) pgs[i] = pl[i];
    __syncwarp();
    auto row = [&](int slot) -> int64_t {
      return base + static_cast<int64_t>(pgs[slot >> lgP]) * pstride + (slot & Pm);
    };
    const bool ranked = ka > tl;
    const int m = ka - tl;
    const int tail_from = n - (ranked ? tl : ka);
    const float *Arow = a.A + (static_cast<int64_t>(l) * a.H + h) * a.max_tokens + a.span[node];
    int ncand = 0;
    for (int s0 = 0; s0 < kc; s0 += 32) {
      const int s = s0 + lane;
      unsigned long long kk = 0;
      if (s < kc) {
        const int p = a.pos[row(s)];
        kk = static_cast<unsigned>(p);
        if (ranked && p < tail_from) {
          const float av = Arow[p];
          if (!(av >= 0.f) || isinf(av)) atomicOr(&a.ctrl->err, DERR_INVARIANT);
          const unsigned bits = (av == 0.f) ? 0u : __float_as_uint(av);   // −0 → +0 (Q3)
          kk = kCand | (static_cast<unsigned long long>(bits) << 16) | static_cast<unsigned>(p);
        }
        key[s] = kk;
      }
      ncand += __popc(__ballot_sync(0xffffffffu, (kk & kCand) != 0));
    }
    __syncwarp();
    unsigned long long tkey = kCand, tmask = kCand;
    if (ranked && m <= 0) {
      tkey = ~0ull; tmask = ~0ull;
    } else if (ranked && m < ncand) {
      unsigned long long prefix = kCand, pmask = kCand;
      int need = m;
      for (int shift = 40; shift >= 0; shift -= 8) {
#pragma unroll
        for (int b = 0; b < 8; ++b) hist[lane * 8 + b] = 0;
        __syncwarp();
        for (int s = lane; s < kc; s += 32) {
          const unsigned long long kk = key[s];
          if ((kk & pmask) == prefix) atomicAdd(&hist[(kk >> shift) & 255u], 1u);
        }
        __syncwarp();
        uint32_t cnt8[8];
        uint32_t loc = 0;
#pragma unroll
        for (int b = 0; b < 8; ++b) { cnt8[b] = hist[255 - lane * 8 - b]; loc += cnt8[b]; }
        uint32_t incl = loc;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
          const uint32_t t = __shfl_up_sync(0xffffffffu, incl, o);
          if (lane >= o) incl += t;
        }
        const uint32_t before = incl - loc;
        const bool mine = before < static_cast<uint32_t>(need) && static_cast<uint32_t>(need) <= incl;
        int dsel = 0;
        uint32_t above = 0, inbin = 0;
        if (mine) {
          uint32_t acc = before;
#pragma unroll
          for (int b = 0; b < 8; ++b) {
            if (inbin == 0 && acc < static_cast<uint32_t>(need) &&
                static_cast<uint32_t>(need) <= acc + cnt8[b]) {
              dsel = 255 - lane * 8 - b;
              above = acc;
              inbin = cnt8[b];
            }
            acc += cnt8[b];
          }
        }
        const int src = __ffs(__ballot_sync(0xffffffffu, mine)) - 1;
        dsel = __shfl_sync(0xffffffffu, dsel, src);
        above = __shfl_sync(0xffffffffu, above, src);
        inbin = __shfl_sync(0xffffffffu, inbin, src);
        need -= static_cast<int>(above);
        prefix |= static_cast<unsigned long long>(dsel) << shift;
        pmask |= 255ull << shift;
        if (static_cast<uint32_t>(need) == inbin) break;
      }
      tkey = prefix;
      tmask = pmask;
    }
    int nh = 0, nm = 0;
    for (int s0 = 0; s0 < kc; s0 += 32) {
      const int s = s0 + lane;
      int keep = 0;
      if (s < kc) {
        const unsigned long long kk = key[s];
        const int p = static_cast<int>(kk & 0xffffu);
        keep = (p >= tail_from) || (ranked && (kk & kCand) && (kk & tmask) >= tkey);
      }
      const int hole = s < ka && !keep;
      const int mv = s >= ka && s < kc && keep;
      const unsigned hb = __ballot_sync(0xffffffffu, hole);
      const unsigned mb = __ballot_sync(0xffffffffu, mv);
      if (hole) holes[nh + __popc(hb & lt_mask)] = s;
      if (mv) movers[nm + __popc(mb & lt_mask)] = s;
      nh += __popc(hb);
      nm += __popc(mb);
    }
    __syncwarp();
    if (nh != nm && lane == 0) atomicOr(&a.ctrl->err, DERR_STATE);
    // hand the job to the move warp
    const int sl = k & 1;
    mbar_wait(&empty[sl], ((k >> 1) & 1) ^ 1);
    int2 *jb = myjobs + sl * jcap;
    for (int i = lane; i < nm; i += 32)
      jb[i] = make_int2(static_cast<int>(row(movers[i])), static_cast<int>(row(holes[i])));
    if (lane == 0) mycount[sl] = nm;
    __syncwarp();
    if (lane == 0) mbar_arrive(&full[sl]);
  }
}

// Move: a pure streaming copy of K, V (rb bytes each) and the pos tag for every listed pair;
// sources and destinations are disjoint, so any order is correct.  cpr lanes per row,
// kUnrollM rows in flight per lane-group.
constexpr int kUnrollM = 4;
__global__ void __launch_bounds__(256, 4)
move_kernel(const Ctrl *__restrict__ ctrl, const int2 *__restrict__ moves, char *__restrict__ kp8,
            char *__restrict__ vp8, int16_t *__restrict__ pos, int rb) {
  const int total = ctrl->move_count;
  const int cpr = rb >> 4;
  const int rpw = 32 / cpr;                    // rows per warp instruction
  const int lane = threadIdx.x & 31;
  const int piece = lane % cpr, sub = lane / cpr;
  const int warps = (gridDim.x * blockDim.x) >> 5;
  const int wg = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int per_iter = rpw * kUnrollM;
  for (int m0 = wg * per_iter; m0 < total; m0 += warps * per_iter) {
    uint4 bk[kUnrollM], bv[kUnrollM];
    int2 mv[kUnrollM];
#pragma unroll
    for (int u = 0; u < kUnrollM; ++u) {
      const int mi = m0 + u * rpw + sub;
      mv[u] = mi < total ? moves[mi] : make_int2(-1, -1);
      if (mv[u].x >= 0) {
        const int64_t off = static_cast<int64_t>(mv[u].x) * rb + piece * 16;
        bk[u] = *reinterpret_cast<const uint4 *>(kp8 + off);
        bv[u] = *reinterpret_cast<const uint4 *>(vp8 + off);
      }
    }
#pragma unroll
    for (int u = 0; u < kUnrollM; ++u) {
      if (mv[u].x >= 0) {
        const int64_t off = static_cast<int64_t>(mv[u].y) * rb + piece * 16;
        *reinterpret_cast<uint4 *>(kp8 + off) = bk[u];
        *reinterpret_cast<uint4 *>(vp8 + off) = bv[u];
        if (piece == 0) pos[mv[u].y] = pos[mv[u].x];
      }
    }
  }
}

}  // namespace

void launch_evict_plan(arbor_ctx *c, int N, const int32_t *k_target) {
  PlanArgs a{};
  a.N = N;
  a.P = c->P;
  a.MPN = c->max_pages_node;
  a.k_target = k_target;
  a.pinned = c->d.pinned;
  a.kcur = c->d.kcur;
  a.npages = c->d.npages;
  a.ptab = c->d.ptab;
  a.free_stack = c->d.free_stack;
  a.work_node = c->d.work_node;
  a.work_old = c->d.work_old;
  a.work_new = c->d.work_new;
  a.ctrl = c->d.ctrl;
  stage_begin(c, ARBOR_ST_EVICT_PLAN, c->ms);
  evict_plan_kernel<<<1, kPlanThreads, 0, c->ms>>>(a);
  ARBOR_LAUNCHED(c);
  stage_end(c, ARBOR_ST_EVICT_PLAN, c->ms);
}

void launch_select_compact(arbor_ctx *c, int max_n) {
  CompactArgs a{};
  a.R = c->L * c->H;
  a.H = c->H;
  a.P = c->P;
  a.D = c->D;
  a.NP = c->NP;
  a.MPN = c->max_pages_node;
  a.l_tail = c->prm.l_tail;
  a.max_tokens = c->max_tokens;
  a.work_node = c->d.work_node;
  a.work_old = c->d.work_old;
  a.work_new = c->d.work_new;
  a.n = c->d.n;
  a.span = c->d.span;
  a.A = c->cfg.score;
  a.ctrl_ro = c->d.ctrl;
  a.ctrl = c->d.ctrl;
  a.ptab = c->d.ptab;
  a.kpool = c->cfg.k_pool;
  a.vpool = c->cfg.v_pool;
  a.pos = c->cfg.pos_pool;
  a.moves = c->d.moves;
  a.esize = c->esize;
  const int cap = max_n < 1 ? 1 : max_n;
  a.cap = cap;
  a.lgP = __builtin_ctz(static_cast<unsigned>(c->P));
  const size_t smem = (static_cast<size_t>(cap) * (8 + 8) + ((cap >> a.lgP) + 1) * 4) * kWarps;
  static size_t attr_smem = 0;
  if (smem > attr_smem) {
    cudaFuncSetAttribute(select_kernel<true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         static_cast<int>(smem < 48 * 1024 ? 48 * 1024 : smem));
    cudaFuncSetAttribute(select_kernel<false>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         static_cast<int>(smem < 48 * 1024 ? 48 * 1024 : smem));
    attr_smem = smem < 48 * 1024 ? 48 * 1024 : smem;
  }
  int sms = 148;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  int per_sm = 0;
  if (kWarpSpecialised) {
    const int jcap = cap / 2 + 1;
    const int pcap = (cap >> a.lgP) + 1;
    const size_t wsm = static_cast<size_t>(kPairs) * cap * (8 + 8) +
                       static_cast<size_t>(((kPairs * pcap + 1) & ~1)) * 4 +
                       static_cast<size_t>(kPairs) * 2 * jcap * 8 + ((kPairs * 2 + 1) & ~1) * 4 +
                       kPairs * 4 * 8;
    static size_t wattr = 0;
    if (wsm > wattr) {
      cudaFuncSetAttribute(select_move_ws_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                           static_cast<int>(wsm < 48 * 1024 ? 48 * 1024 : wsm));
      wattr = wsm < 48 * 1024 ? 48 * 1024 : wsm;
    }
    int per = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, select_move_ws_kernel, kPairs * 64, wsm);
    stage_begin(c, ARBOR_ST_SELECT_COMPACT, c->ms);
    select_move_ws_kernel<<<sms * (per > 0 ? per : 1), kPairs * 64, wsm, c->ms>>>(a);
    ARBOR_LAUNCHED(c);
    stage_end(c, ARBOR_ST_SELECT_COMPACT, c->ms);
    return;
  }
  const bool fused = kFusedCompact;
  if (fused) cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, select_kernel<true>, kWarps * 32, smem);
  else cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, select_kernel<false>, kWarps * 32, smem);
  stage_begin(c, ARBOR_ST_SELECT_COMPACT, c->ms);
  if (fused) select_kernel<true><<<sms * (per_sm > 0 ? per_sm : 1), kWarps * 32, smem, c->ms>>>(a);
  else select_kernel<false><<<sms * (per_sm > 0 ? per_sm : 1), kWarps * 32, smem, c->ms>>>(a);
  ARBOR_LAUNCHED(c);
  stage_end(c, ARBOR_ST_SELECT_COMPACT, c->ms);
  if (fused) return;
  int per_sm_m = 0;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm_m, move_kernel, 256, 0);
  stage_begin(c, ARBOR_ST_COMPACT_MOVE, c->ms);
  move_kernel<<<sms * (per_sm_m > 0 ? per_sm_m : 1), 256, 0, c->ms>>>(
      c->d.ctrl, c->d.moves, static_cast<char *>(c->cfg.k_pool), static_cast<char *>(c->cfg.v_pool),
      c->cfg.pos_pool, c->D * c->esize);
  ARBOR_LAUNCHED(c);
  stage_end(c, ARBOR_ST_COMPACT_MOVE, c->ms);
}

}  // namespace arbor
