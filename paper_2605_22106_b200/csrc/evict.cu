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
constexpr int kPairsWs = 8;   // (select warp, move warp) pairs per CTA of select_move_ws_kernel
constexpr int kUw = 4;        // rows in flight per lane group of a move warp

struct PlanArgs {
  int N, P, MPN;
  const int32_t *k_target;
  const uint8_t *pinned;
  int32_t *kcur, *npages, *ptab, *free_stack;
  const int32_t *n;
  const int64_t *span;
  WorkEnt *work;
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
    WorkEnt e;
    e.node = j;
    e.kc = kc[i];
    e.ka = kapp[i];
    e.n = a.n[j];
    e.span = a.span[j];
    e.pad = 0;
    a.work[work_off] = e;
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
  const WorkEnt *work;
  const float *A;
  const Ctrl *ctrl_ro;
  Ctrl *ctrl;
  const int32_t *ptab;
  void *kpool, *vpool;
  int16_t *pos;
  int esize;
  int cap;          // max n over evicted nodes (smem capacity, slots)
  int lgP;          // log2(page size)
  int exp;          // ARBOR_EVICT_EXP (measurement only): bit0 skip moves, bit1 skip radix select
};

__device__ __forceinline__ void cp_async4(void *smem, const void *gmem) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 4;\n" ::"r"(smem_u32(smem)), "l"(gmem)
               : "memory");
}
__device__ __forceinline__ void cp_async16ca(void *smem, const void *gmem) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 16;\n" ::"r"(smem_u32(smem)), "l"(gmem)
               : "memory");
}

// Shared-memory layout of select_move_ws_kernel (per CTA), all offsets 16-byte aligned.
struct WsLayout {
  int cap, capP, pcap, jcap;
  size_t keys, lists, abuf, pbuf, gbuf, mbuf, jobs, jcount, bars, total;
  __host__ __device__ WsLayout(int cap_, int lgP) {
    cap = cap_;
    capP = (cap + 9) & ~7;                 // pos pairs may read one slot past k_cur
    pcap = (cap >> lgP) + 2;
    jcap = cap / 2 + 1;                    // moves per item ≤ min(k_app, k_cur − k_app)
    size_t o = 0;
    auto take = [&](size_t bytes) { size_t r = o; o += (bytes + 15) & ~size_t(15); return r; };
    keys = take(size_t(kPairsWs) * cap * 8);              // u64 keys
    lists = take(size_t(kPairsWs) * 2 * cap * 4);         // holes | movers
    abuf = take(size_t(kPairsWs) * 2 * cap * 4);          // A span, 2 pipeline slots
    pbuf = take(size_t(kPairsWs) * 2 * capP * 2);         // pos tags, 2 pipeline slots
    gbuf = take(size_t(kPairsWs) * 3 * pcap * 4);         // page lists, 3 pipeline slots
    mbuf = take(size_t(kPairsWs) * 4 * sizeof(WorkEnt));  // work entries, 4 pipeline slots
    jobs = take(size_t(kPairsWs) * 2 * jcap * 8);         // (src row, dst row) job queues
    jcount = take(size_t(kPairsWs) * 2 * 4);
    bars = take(size_t(kPairsWs) * 4 * 8);
    total = o;
  }
};

// Warp-specialised select + move.  A CTA holds kPairsWs (select warp, move warp) pairs.
//
// Select warp p processes the work items it = first + k·stride (item = (changed node, row)).
// Its global reads run three items ahead through a cp.async pipeline (no register cost, no
// exposed latency): work entry of item k+3 → page list of item k+2 → pos tags and A span of
// item k+1 (A is read by position over the span, independent of the pos tags), while item k
// is ranked from shared memory.  Keep = the block tail 𝒯 (positions ≥ n − |𝒯|)
// ∪ the top-m non-tail candidates by the 48-bit key ⟨A bits, pos⟩, or the last
// k_app positions when k_app ≤ |𝒯| (Alg. 1).  The m-th largest key is found by a
// warp radix select (8-bit digits, per-warp smem histogram, warp scan) that starts at the
// highest key bit on which the candidates differ (warp min/max reductions of the A bits), so
// the shared exponent bits cost no pass.  Slot layout (Q23'): kept rows in slots
// [0, k_app) stay; the i-th hole there takes the i-th kept row from slots ≥ k_app.  The item's
// (src row, dst row) list goes to move warp p through a 2-slot job queue in shared memory
// guarded by mbarriers (full / empty).
//
// Move warp p streams those rows (K, V: 16-byte coalesced, kUw rows in flight per lane group;
// pos tags).  Sources and destinations are disjoint, so moves need no ordering.
__global__ void __launch_bounds__(kPairsWs * 64, 2)
select_move_ws_kernel(CompactArgs a) {
  extern __shared__ __align__(16) unsigned char sm[];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const bool mover = warp >= kPairsWs;
  const int pid = mover ? warp - kPairsWs : warp;
  const WsLayout Ly(a.cap, a.lgP);
  const int cap = Ly.cap, capP = Ly.capP, pcap = Ly.pcap, jcap = Ly.jcap;
  const int lgP = a.lgP, Pm = (1 << lgP) - 1;
  uint64_t *bars = reinterpret_cast<uint64_t *>(sm + Ly.bars);
  uint64_t *full = bars + pid * 4, *empty = bars + pid * 4 + 2;
  int2 *myjobs = reinterpret_cast<int2 *>(sm + Ly.jobs) + pid * 2 * jcap;
  int32_t *mycount = reinterpret_cast<int32_t *>(sm + Ly.jcount) + pid * 2;
  __shared__ uint32_t hist_all[kPairsWs][256];
  if (threadIdx.x == 0) {
    for (int i = 0; i < kPairsWs * 2; ++i) {
      mbar_init(&bars[(i >> 1) * 4 + (i & 1)], 1);
      mbar_init(&bars[(i >> 1) * 4 + 2 + (i & 1)], 1);
    }
    mbar_fence_init();
  }
  __syncthreads();
  const int items = a.ctrl_ro->work_count * a.R;
  const int stride = gridDim.x * kPairsWs;
  const int first = blockIdx.x * kPairsWs + pid;
  if (mover) {
    // ------------------------------------------------------------ move warp
    const int rb = a.D * a.esize, cpr = rb >> 4, rpi = 32 / cpr;
    const int piece = lane % cpr, sub = lane / cpr;
    char *kp8 = static_cast<char *>(a.kpool);
    char *vp8 = static_cast<char *>(a.vpool);
    int k = 0;
    for (int it = first; it < items; it += stride, ++k) {
      const int sl = k & 1;
      mbar_wait(&full[sl], (k >> 1) & 1);
      const int nm = (a.exp & 1) ? 0 : mycount[sl];
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
  unsigned long long *key = reinterpret_cast<unsigned long long *>(sm + Ly.keys) + pid * cap;
  int32_t *holes = reinterpret_cast<int32_t *>(sm + Ly.lists) + pid * 2 * cap;
  int32_t *movers = holes + cap;
  float *Abuf = reinterpret_cast<float *>(sm + Ly.abuf) + pid * 2 * cap;
  int16_t *Pbuf = reinterpret_cast<int16_t *>(sm + Ly.pbuf) + pid * 2 * capP;
  int32_t *Gbuf = reinterpret_cast<int32_t *>(sm + Ly.gbuf) + pid * 3 * pcap;
  WorkEnt *Mbuf = reinterpret_cast<WorkEnt *>(sm + Ly.mbuf) + pid * 4;
  uint32_t *hist = hist_all[pid];
  const unsigned lt_mask = (1u << lane) - 1u;
  const int64_t pstride = static_cast<int64_t>(a.H) << lgP;
  constexpr unsigned long long kCand = 1ull << 63;
  const int my_items = first < items ? (items - first + stride - 1) / stride : 0;
  auto row_base = [&](int it) -> int64_t {
    const int r = it % a.R;
    const int l = r / a.H, h = r - l * a.H;
    return (static_cast<int64_t>(l) * a.NP * a.H + h) << lgP;
  };
  // pipeline stages (each lane issues its share; completion via cp.async.wait_all + __syncwarp)
  auto issue_meta = [&](int k) {
    if (k >= my_items || lane >= 2) return;
    const int w = (first + k * stride) / a.R;
    cp_async16ca(reinterpret_cast<char *>(&Mbuf[k & 3]) + lane * 16,
                 reinterpret_cast<const char *>(&a.work[w]) + lane * 16);
  };
  auto issue_pages = [&](int k) {
    if (k >= my_items) return;
    const WorkEnt &e = Mbuf[k & 3];
    const int np = (e.kc + Pm) >> lgP;
    const int32_t *pl = a.ptab + static_cast<int64_t>(e.node) * a.MPN;
    int32_t *g = Gbuf + (k % 3) * pcap;
    for (int i = lane; i < np; i += 32) cp_async4(g + i, pl + i);
  };
  auto issue_data = [&](int k) {
    if (k >= my_items) return;
    const int it = first + k * stride;
    const WorkEnt &e = Mbuf[k & 3];
    const int32_t *g = Gbuf + (k % 3) * pcap;
    const int64_t base = row_base(it);
    int16_t *pb = Pbuf + (k & 1) * capP;
    for (int q = lane; 2 * q < e.kc; q += 32) {     // slot pairs (P even: same page)
      const int s = 2 * q;
      cp_async4(pb + s, a.pos + base + static_cast<int64_t>(g[s >> lgP]) * pstride + (s & Pm));
    }
    const int tl = min(a.l_tail, e.n);
    if (e.ka > tl) {               // ranked: A of the non-tail positions
      const int r = it % a.R;
      const float *Arow = a.A + static_cast<int64_t>(r) * a.max_tokens + e.span;
      float *ab = Abuf + (k & 1) * cap;
      for (int p = lane; p < e.n - tl; p += 32) cp_async4(ab + p, Arow + p);
    }
  };
  if (my_items > 0) {
    issue_meta(0);
    cp_async_commit();
    cp_async_wait_all();
    __syncwarp();
    issue_pages(0);
    issue_meta(1);
    cp_async_commit();
    cp_async_wait_all();
    __syncwarp();
    issue_data(0);
    issue_pages(1);
    issue_meta(2);
    cp_async_commit();
  }
  for (int k = 0; k < my_items; ++k) {
    cp_async_wait_all();
    __syncwarp();
    issue_data(k + 1);
    issue_pages(k + 2);
    issue_meta(k + 3);
    cp_async_commit();
    // ---- rank item k from shared memory
    const int it = first + k * stride;
    const WorkEnt e = Mbuf[k & 3];
    const int kc = e.kc, ka = e.ka, n = e.n;
    const int tl = min(a.l_tail, n);
    const int32_t *pgs = Gbuf + (k % 3) * pcap;
    const int16_t *pb = Pbuf + (k & 1) * capP;
    const float *ab = Abuf + (k & 1) * cap;
    const int64_t base = row_base(it);
    auto row = [&](int slot) -> int64_t {
      return base + static_cast<int64_t>(pgs[slot >> lgP]) * pstride + (slot & Pm);
    };
    const bool ranked = ka > tl;
    const int m = ka - tl;
    const int tail_from = n - (ranked ? tl : ka);   // keep positions ≥ tail_from outright
    int ncand = 0;
    uint32_t bmin = 0xffffffffu, bmax = 0u;
    for (int s0 = 0; s0 < kc; s0 += 32) {
      const int s = s0 + lane;
      unsigned long long kk = 0;
      if (s < kc) {
        const int p = pb[s];
        kk = static_cast<unsigned>(p);
        if (ranked && p < tail_from) {
          const float av = ab[p];
          if (!(av >= 0.f) || isinf(av)) atomicOr(&a.ctrl->err, DERR_INVARIANT);
          const unsigned bits = (av == 0.f) ? 0u : __float_as_uint(av);   // −0 → +0 (Q3)
          kk = kCand | (static_cast<unsigned long long>(bits) << 16) | static_cast<unsigned>(p);
          bmin = min(bmin, bits);
          bmax = max(bmax, bits);
        }
        key[s] = kk;
      }
      ncand += __popc(__ballot_sync(0xffffffffu, (kk & kCand) != 0));
    }
    __syncwarp();
    // threshold: keep a candidate iff (key & tmask) >= tkey (the top m unique keys)
    unsigned long long tkey = kCand, tmask = kCand;     // m ≥ ncand: all candidates
    if (ranked && m <= 0) {
      tkey = ~0ull; tmask = ~0ull;                      // none survives
    } else if (ranked && m < ncand && !(a.exp & 2)) {
      // candidates share every key bit above `top` (bits of A above the highest bit where
      // min and max differ); the radix passes start there
      bmin = __reduce_min_sync(0xffffffffu, bmin);
      bmax = __reduce_max_sync(0xffffffffu, bmax);
      const int top = bmin != bmax ? 16 + 31 - __clz(static_cast<int>(bmin ^ bmax)) : 15;
      unsigned long long prefix = kCand, pmask = kCand;
      int need = m;
      for (int shift = top - 7; shift > -8; shift -= 8) {
        const unsigned long long dmask = shift >= 0 ? 255ull << shift : 255ull >> -shift;
#pragma unroll
        for (int b = 0; b < 8; ++b) hist[lane * 8 + b] = 0;
        __syncwarp();
        for (int s = lane; s < kc; s += 32) {
          const unsigned long long kk = key[s];
          if ((kk & pmask) == prefix) {
            const unsigned dg = shift >= 0 ? static_cast<unsigned>(kk >> shift) & 255u
                                           : static_cast<unsigned>(kk << -shift) & 255u;
            atomicAdd(&hist[dg], 1u);
          }
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
        prefix |= shift >= 0 ? static_cast<unsigned long long>(dsel) << shift
                             : static_cast<unsigned long long>(dsel) >> -shift;
        pmask |= dmask;
        if (static_cast<uint32_t>(need) == inbin) break;   // the whole bin survives
      }
      tkey = prefix;
      tmask = pmask;
    }
    // keep flags → holes (dropped slots < k_app) and movers (kept slots ≥ k_app), ascending
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
    if (nh != nm && lane == 0 && !a.exp) atomicOr(&a.ctrl->err, DERR_STATE);
    if (a.exp) nm = nm < nh ? nm : nh;
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
  a.n = c->d.n;
  a.span = c->d.span;
  a.work = c->d.work;
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
  a.work = c->d.work;
  a.A = c->cfg.score;
  a.ctrl_ro = c->d.ctrl;
  a.ctrl = c->d.ctrl;
  a.ptab = c->d.ptab;
  a.kpool = c->cfg.k_pool;
  a.vpool = c->cfg.v_pool;
  a.pos = c->cfg.pos_pool;
  a.esize = c->esize;
  a.cap = max_n < 1 ? 1 : max_n;
  a.lgP = __builtin_ctz(static_cast<unsigned>(c->P));
  static const int exp_flags = [] {
    const char *e = getenv("ARBOR_EVICT_EXP");
    return e ? atoi(e) : 0;
  }();
  a.exp = exp_flags;
  const WsLayout ly(a.cap, a.lgP);
  // occupancy / smem attribute cached per capacity (host-side cost stays off the launch path)
  static size_t attr_smem = 0;
  static int cached_cap = -1, cached_lg = -1, cached_grid = 0;
  if (ly.total > attr_smem) {
    const size_t want = ly.total < 48 * 1024 ? 48 * 1024 : ly.total;
    cudaFuncSetAttribute(select_move_ws_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         static_cast<int>(want));
    attr_smem = want;
  }
  if (a.cap != cached_cap || a.lgP != cached_lg) {
    int sms = 148, per = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, select_move_ws_kernel, kPairsWs * 64, ly.total);
    cached_grid = sms * (per > 0 ? per : 1);
    cached_cap = a.cap;
    cached_lg = a.lgP;
  }
  stage_begin(c, ARBOR_ST_SELECT_COMPACT, c->ms);
  select_move_ws_kernel<<<cached_grid, kPairsWs * 64, ly.total, c->ms>>>(a);
  ARBOR_LAUNCHED(c);
  stage_end(c, ARBOR_ST_SELECT_COMPACT, c->ms);
}

}  // namespace arbor
