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
//    nodes in ascending id, frees the leading pages before the kept window (soff moves up,
//    DESIGN.md Q23*) and pushes them on the LIFO free list nodes ascending, each node's run
//    in descending list order — all on the device, no host sync.
//  * select (persistent grid, one WARP per (node, row) work item, no block barriers):
//    pos tags + A keys of the kept slots, the m-th largest unique 48-bit key ⟨A bits, pos⟩
//    by a warp radix select (8-bit digits, per-warp smem histogram, warp scan) — exact top-m
//    membership in O(c) — then end-window hole filling: the new block is the last k_app
//    valid slots (where the always-kept block tail 𝒯 sits), kept rows inside it stay, the
//    i-th hole takes the i-th kept row from before it (Q23*: ~1/3 fewer moved rows
//    than a [0, k_app) prefix on C2).  Sources and destinations are disjoint.
//  * move (persistent grid): a pure 16-byte-coalesced streaming copy of the listed K, V
//    rows and pos tags — no ordering constraints, full occupancy.
#include <type_traits>
#include <cub/block/block_scan.cuh>

#include "tile.cuh"

namespace arbor {
namespace {

#ifndef ARBOR_PAIRS
#define ARBOR_PAIRS 8
#endif
constexpr int kPairsWs = ARBOR_PAIRS;   // (select warp, move warp) pairs per CTA of select_move_ws_kernel
#ifndef ARBOR_KUW
#define ARBOR_KUW 4
#endif
constexpr int kUw = ARBOR_KUW;   // rows in flight per lane group of a move warp
#ifndef ARBOR_JOB_SLOTS
#define ARBOR_JOB_SLOTS 2
#endif
#ifndef ARBOR_EVICT_SLEEP_NS
#define ARBOR_EVICT_SLEEP_NS 2000
#endif
constexpr int kJobSlots = ARBOR_JOB_SLOTS;   // job queue depth per pair (power of 2; 2, 4, 8 measured equal on C2)
static_assert((kJobSlots & (kJobSlots - 1)) == 0, "job slots: a power of two");

struct CompactArgs {
  int R;            // rows = L * H
  int H, P, D, NP, MPN, l_tail;
  int64_t max_tokens;
  WorkEnt *work;    // [grid][max_nodes]: each CTA's private copy of the work list
  int N, MN;        // tree nodes, max_nodes (work-list stride)
  const int32_t *k_target, *n;
  const uint8_t *pinned;
  const int64_t *span;
  int32_t *kcur, *npages, *free_stack;
  int32_t *soff;    // page-list slot of each node's valid slot 0 (Q23*)
  const float *A;
  const float *Ahat;   // select_shared: the slice-summed Â[t] every row ranks by (else NULL)
  const Ctrl *ctrl_ro;
  Ctrl *ctrl;
  const int32_t *ptab;
  void *kpool, *vpool;
  int16_t *pos;
  int esize;
  int cap;          // max n over evicted nodes (smem capacity, slots)
  int lgP;          // log2(page size)
  int exp;          // ARBOR_EVICT_EXP (measurement only): bit0 skip moves, bit1 skip radix select
  int select_mode;  // arbor_select_mode (f4)
  int n_sinks;      // global sinks: the root's first n_sinks positions (HEAVY, SINKS_TAIL)
  long long *trace; // ARBOR_EVICT_TRACE=1 (diagnostics): [cta][warp][4] globaltimer ns
  int wl_smem;      // N when the work list also lives in shared memory (N ≤ kSmemWorkNodes), else 0
  const int32_t *gate;   // f1 device waterline: nothing to do when *gate == 0 (else NULL)
};
constexpr int kSmemWorkNodes = 1024;   // 32 KB of work entries per CTA
#ifndef ARBOR_FINISH
#define ARBOR_FINISH 32
#endif
constexpr int kFinish = ARBOR_FINISH;   // ≤ 32; radix passes stop once this few keys share the prefix (rank-count finish)
// slot loops of the select warp are kept rolled: unrolling them 2x / 4x measured slower (C5
// select_compact 278 -> 294-296 us; C2 113 -> 114-115 us), as did the compiler's default
constexpr int kSelUnroll = 1;
// … except the hole / mover list build: unrolled 4x it measured C2 113.4 -> 112.2 us, C5
// 278.3 -> 276.7 us (the key build unrolled alone: C5 300 us; hoisting its uniform tests and
// deferring its invariant check out of the loop: C5 287 us — register pressure at the cap)
#ifndef ARBOR_UNROLL_LISTS
#define ARBOR_UNROLL_LISTS 4
#endif
constexpr int kUnrollLists = ARBOR_UNROLL_LISTS;

__device__ __forceinline__ long long gtimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return static_cast<long long>(t);
}
constexpr int kTraceSlots = 16;
// the timeline (ARBOR_EVICT_TRACE=1 at run time) is compiled only into diagnostic builds
// (-DARBOR_EVICT_TRACE_BUILD): its clock reads and counters cost the production kernel
// registers at its 64-register cap
#ifdef ARBOR_EVICT_TRACE_BUILD
constexpr bool kTrace = true;
#else
constexpr bool kTrace = false;
#endif
// the isolation experiments (ARBOR_EVICT_EXP at run time: skip moves / the radix select) are
// compiled only into -DARBOR_EVICT_EXP_BUILD builds, for the same reason
#ifdef ARBOR_EVICT_EXP_BUILD
constexpr bool kExp = true;
#else
constexpr bool kExp = false;
#endif   // per warp: 8 events / counters + 8 select-phase cycle sums
// select-phase cycle sums (debug builds with -DARBOR_EVICT_PHASES, trace slots 8-13): 5 the
// cp.async wait for the item's data, 0 the next items' issues, 1 key build, 2 threshold,
// 3 hole / mover lists, 4 job hand-off; slot 14: items
#ifdef ARBOR_EVICT_PHASES
#define PH_MARK(i)                                      \
  do {                                                  \
    if (kTrace && a.trace) {                            \
      const long long t_ = clock64();                   \
      ph[i] += t_ - ph_t;                               \
      ph_t = t_;                                        \
    }                                                   \
  } while (0)
#else
#define PH_MARK(i) do { } while (0)
#endif
// trace events per warp: 0 kernel start (after griddepcontrol.wait), 1 plan done,
// 2 first job handed / started, 3 last job handed / done, 4 plan loads done, 5 plan scans done
#define EV_TRACE(e)                                                                           \
  do {                                                                                        \
    if (kTrace && a.trace && lane == 0)                                                                 \
      a.trace[(static_cast<int64_t>(blockIdx.x) * (2 * kPairsWs) + warp) * kTraceSlots + (e)] = gtimer(); \
  } while (0)


__device__ __forceinline__ void cp_async4(void *smem, const void *gmem) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 4;\n" ::"r"(smem_u32(smem)), "l"(gmem)
               : "memory");
}
__device__ __forceinline__ void cp_async16ca(void *smem, const void *gmem) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 16;\n" ::"r"(smem_u32(smem)), "l"(gmem)
               : "memory");
}

// Streams nm (src row, dst row) pairs — K and V rows 16-byte coalesced (a row is cpr lanes,
// rpi rows per warp instruction, U instructions in flight per lane), pos tags by the lane
// holding piece 0.  src(i) / dst(i) give the rows of pair i.  Sources and destinations are
// disjoint (Q23'), so the pairs need no order.
template <int U, typename Src, typename Dst>
__device__ __forceinline__ void move_rows(int nm, Src src, Dst dst, char *kp8, char *vp8,
                                          int16_t *pos, int rb, int rpi, int piece, int sub) {
  for (int c0 = 0; c0 < nm; c0 += rpi * U) {
    uint4 bk[U], bv[U];
    int sr[U], dr[U];
    int16_t pt[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int i = c0 + u * rpi + sub;
      sr[u] = i < nm ? src(i) : -1;
      dr[u] = i < nm ? dst(i) : -1;
      if (sr[u] >= 0) {
        const int64_t off = static_cast<int64_t>(sr[u]) * rb + piece * 16;
        bk[u] = *reinterpret_cast<const uint4 *>(kp8 + off);
        bv[u] = *reinterpret_cast<const uint4 *>(vp8 + off);
        if (piece == 0) pt[u] = pos[sr[u]];
      }
    }
#pragma unroll
    for (int u = 0; u < U; ++u) {
      if (sr[u] >= 0) {
        const int64_t off = static_cast<int64_t>(dr[u]) * rb + piece * 16;
        *reinterpret_cast<uint4 *>(kp8 + off) = bk[u];
        *reinterpret_cast<uint4 *>(vp8 + off) = bv[u];
        if (piece == 0) pos[dr[u]] = pt[u];
      }
    }
  }
}

// Shared-memory layout of select_move_ws_kernel (per CTA), all offsets 16-byte aligned.
struct WsLayout {
  int cap, capA, capP, pcap, jcap;
  int wl_n;                                // nodes of the shared-memory work list (0: global)
  size_t keys, lists, abuf, pbuf, gbuf, mbuf, jobs, jcount, bars, iring, swl, total;
  __host__ __device__ WsLayout(int cap_, int lgP, int wl_n_) {
    cap = cap_;
    wl_n = wl_n_;
    capA = (cap + 9) & ~3;                 // A span from its 16-byte-aligned start (≤ 3 floats before)
    capP = (cap + (1 << lgP) + 9) & ~7;   // pos tags by page-list slot from soff mod P (+1: pairs)
    pcap = (cap >> lgP) + 2;
    jcap = cap / 2 + 1;                    // moves per item ≤ min(k_app, k_cur − k_app)
    size_t o = 0;
    auto take = [&](size_t bytes) { size_t r = o; o += (bytes + 15) & ~size_t(15); return r; };
    keys = take(size_t(kPairsWs) * cap * 8);              // u64 keys
    lists = take(size_t(kPairsWs) * 2 * cap * 4);         // holes | movers
    abuf = take(size_t(kPairsWs) * 2 * capA * 4);         // A span, 2 pipeline slots
    pbuf = take(size_t(kPairsWs) * 2 * capP * 2);         // pos tags, 2 pipeline slots
    gbuf = take(size_t(kPairsWs) * 3 * pcap * 4);         // page lists, 3 pipeline slots
    mbuf = take(size_t(kPairsWs) * 4 * sizeof(WorkEnt));  // work entries, 4 pipeline slots
    jobs = take(size_t(kPairsWs) * kJobSlots * jcap * 8);  // (src row, dst row) job queues
    jcount = take(size_t(kPairsWs) * kJobSlots * 4);
    bars = take(size_t(kPairsWs) * 2 * kJobSlots * 8);
    iring = take(size_t(kPairsWs) * 4 * 4 * 2);            // drawn work items + their work entries
    swl = take(size_t(wl_n) * sizeof(WorkEnt));            // this CTA's work list (small trees)
    total = o;
  }
};

// Warp-specialised select + move.  A CTA holds kPairsWs (select warp, move warp) pairs.
//
// Select warp p processes work items (item = (changed node, row)) drawn from a global counter.
// Its global reads run ahead through a cp.async pipeline (no register cost, no exposed
// latency): work entry of item k+3 (global work list only) → page list of item k+2 → pos tags and A span of
// item k+1 (A is read by position over the span, independent of the pos tags), while item k
// is ranked from shared memory.  Keep = the block tail 𝒯 (positions ≥ n − |𝒯|)
// ∪ the top-m non-tail candidates by the 49-bit key ⟨sink, A bits, pos⟩,
// or the last k_app positions when k_app ≤ |𝒯| (Alg. 1).  The m-th largest key is
// found by a warp radix select (8-bit digits, per-warp smem histogram, warp scan) that starts
// at the highest key bit on which the candidates differ (warp min/max reductions), so the
// shared exponent bits cost no pass.  Slot layout (Q23*): the new block is the
// window of the last k_app valid slots; kept rows there stay, the i-th hole there takes the
// i-th kept row from before the window.  The item's
// (src row, dst row) list goes to move warp p through a 2-slot job queue in shared memory
// guarded by mbarriers (full / empty).
//
// Move warp p streams those rows (K, V: 16-byte coalesced, kUw rows in flight per lane group;
// pos tags).  Sources and destinations are disjoint, so moves need no ordering.
// CAPT > 0: a compile-time capacity (k_cur ≤ CAPT) and page size 2^LGPT — every shared-memory
// offset of the layout is then a constant off one base address, which at the 64-register cap
// saves the registers (and the rematerialisation) that runtime offsets cost; CAPT = 0: runtime
template <int CAPT, int LGPT, int HT>
__global__ void __launch_bounds__(kPairsWs * 64, 2)
select_move_ws_kernel(CompactArgs a) {
  const int H = HT ? HT : a.H;           // KV heads of a row index (a constant divisor when HT > 0)
  extern __shared__ __align__(16) unsigned char sm[];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const bool mover = warp >= kPairsWs;
  const int pid = mover ? warp - kPairsWs : warp;
  const WsLayout Ly(CAPT ? CAPT : a.cap, CAPT ? LGPT : a.lgP, a.wl_smem);
  const int cap = Ly.cap, capA = Ly.capA, capP = Ly.capP, pcap = Ly.pcap, jcap = Ly.jcap;
  const int lgP = CAPT ? LGPT : a.lgP, Pm = (1 << lgP) - 1;
  uint64_t *bars = reinterpret_cast<uint64_t *>(sm + Ly.bars);
  uint64_t *full = bars + pid * 2 * kJobSlots, *empty = full + kJobSlots;
  int2 *myjobs = reinterpret_cast<int2 *>(sm + Ly.jobs) + pid * kJobSlots * jcap;
  int32_t *mycount = reinterpret_cast<int32_t *>(sm + Ly.jcount) + pid * kJobSlots;
  __shared__ __align__(16) uint32_t hist_all[kPairsWs][256];
  using Scan = cub::BlockScan<int, kPairsWs * 64>;
  __shared__ typename Scan::TempStorage scan_tmp;
  __shared__ int s_work, s_free, s_apply;
  __shared__ unsigned long long s_ev;
  if (threadIdx.x == 0) {
    for (int i = 0; i < kPairsWs * 2 * kJobSlots; ++i) mbar_init(&bars[i], 1);
    mbar_fence_init();
    s_ev = 0;
  }
  __syncthreads();
  pdl_wait();
  pdl_trigger();
  if (a.gate && *a.gate == 0) return;   // the waterline did not fire: k = k_cur everywhere
  EV_TRACE(0);
  // ---- plan (Alg. 2, Q17): k_app = min(k_cur, k_target) for every non-pinned node;
  // the changed ones, ascending id, are the work list.  Every CTA derives it from the same
  // unmodified state into its own copy; the last CTA to get there (ticket) applies it —
  // k_cur, page-list truncation to ⌈k_app/P⌉, freed pages pushed on the LIFO free stack in
  // ascending node order (each node's run descending) — after every CTA has read that state.
  WorkEnt *wl = a.work + static_cast<int64_t>(blockIdx.x) * a.MN;
  {
    // nodes j = i·blockDim + thread, one slice i at a time: the slice's loads in one round
    // trip, then two block scans (work list offsets, freed-page offsets) in ascending id;
    // most trees (N ≤ blockDim) are a single slice
    int tot_work = 0, tot_free = 0;
    unsigned long long my_ev = 0;
    WorkEnt *swl = reinterpret_cast<WorkEnt *>(sm + Ly.swl);
    for (int j0 = 0; j0 < a.N; j0 += blockDim.x) {
      const int j = j0 + threadIdx.x;
      int kc = 0, kt = 0, nn = 0, npg = 0, so = 0;
      long long sp = 0;
      bool pin = true;
      if (j < a.N) {
        kc = a.kcur[j];
        kt = a.k_target[j];
        pin = a.pinned[j] != 0;
        npg = a.npages[j];
        nn = a.n[j];
        sp = a.span[j];
        so = a.soff[j];
      }
      const int ka = min(max(kt, 0), kc);
      const int ev = (!pin && ka < kc) ? 1 : 0;
      if (j0 == 0) EV_TRACE(4);
      // freed: the live pages before the one holding the window's first slot so + kc − ka
      // (every live page when nothing is kept)
      const int fr = ev ? (ka > 0 ? ((so + kc - ka) >> lgP) : npg) - (so >> lgP) : 0;
      if (ev) my_ev += static_cast<unsigned long long>(kc - ka);
      int wo, fo, tw, tf;
      Scan(scan_tmp).ExclusiveSum(ev, wo, tw);
      __syncthreads();
      Scan(scan_tmp).ExclusiveSum(fr, fo, tf);
      __syncthreads();
      if (j0 == 0) EV_TRACE(5);
      if (ev) {
        WorkEnt e;
        e.node = j;
        e.kc = kc;
        e.ka = ka;
        e.n = nn;
        e.span = sp;
        e.foff = tot_free + fo;
        e.nfree = static_cast<int16_t>(fr);
        e.so = static_cast<int16_t>(so);
        wl[tot_work + wo] = e;
        if (Ly.wl_n) swl[tot_work + wo] = e;
      }
      tot_work += tw;
      tot_free += tf;
    }
    // evicted-token count: warp sums first — one 64-bit shared atomic per thread (156 on C2)
    // serialised into ~3-8 µs of the plan (evict_trace: scans done at 1.8 µs, plan at 7.9)
#pragma unroll
    for (int o = 16; o; o >>= 1) my_ev += __shfl_xor_sync(0xffffffffu, my_ev, o);
    if (lane == 0 && my_ev) atomicAdd(&s_ev, my_ev);
    if (threadIdx.x == 0) { s_work = tot_work; s_free = tot_free; }
  }
  __syncthreads();
  EV_TRACE(1);
  const int items = s_work * a.R;
  if (mover) {
    // the move warps take the ticket (they would otherwise wait for their first job)
    const int mt = threadIdx.x - kPairsWs * 32;
    if (mt == 0) {
      __threadfence();
      const unsigned t = atomicAdd(reinterpret_cast<unsigned *>(&a.ctrl->plan_ticket), 1u);
      s_apply = t == gridDim.x - 1;
    }
    named_bar_sync(1, kPairsWs * 32);
    if (s_apply) {
      __threadfence();
      const int top = a.ctrl->free_top;
      for (int w = mt; w < s_work; w += kPairsWs * 32) {
        const WorkEnt e = wl[w];
        const int32_t *__restrict__ pl = a.ptab + static_cast<int64_t>(e.node) * a.MPN + (e.so >> lgP);
        int32_t *__restrict__ dst = a.free_stack + top + e.foff;
        constexpr int kB = 8;
        for (int t0 = 0; t0 < e.nfree; t0 += kB) {
          int32_t v[kB];
#pragma unroll
          for (int t = 0; t < kB; ++t) v[t] = t0 + t < e.nfree ? __ldg(pl + t0 + t) : 0;
#pragma unroll
          // descending list order (Q23''): LIFO pops return the run ascending
          for (int t = 0; t < kB; ++t) if (t0 + t < e.nfree) dst[e.nfree - 1 - (t0 + t)] = v[t];
        }
        // the window's page-list slots stay where they are: soff moves up, the stale
        // entries below it are never read again (an empty node resets)
        if (e.ka > 0) {
          a.soff[e.node] = e.so + e.kc - e.ka;
        } else {
          a.soff[e.node] = 0;
          a.npages[e.node] = 0;
        }
        a.kcur[e.node] = e.ka;
      }
      if (mt == 0) {
        a.ctrl->free_top = top + s_free;
        a.ctrl->work_count = s_work;
        a.ctrl->evicted = static_cast<long long>(s_ev);
        a.ctrl->pages_in_use -= s_free;
        a.ctrl->plan_ticket = 0;
      }
    }
    // ------------------------------------------------------------ move warp
    const int rb = a.D * a.esize, cpr = rb >> 4, rpi = 32 / cpr;
    const int piece = lane % cpr, sub = lane / cpr;
    char *kp8 = static_cast<char *>(a.kpool);
    char *vp8 = static_cast<char *>(a.vpool);
    // jobs until the select warp posts the end marker (count < 0): the items are handed out
    // dynamically, so the number of jobs is not known in advance
    long long mv_rows = 0, w_full = 0;
    int k_jobs = 0;
    for (int k = 0;; ++k) {
      const int sl = k & (kJobSlots - 1);
      const long long tw0 = (kTrace && a.trace) ? clock64() : 0;
      // a starved move warp sleeps in the try_wait instead of spinning: its spin loop took
      // ~18% of the kernel's issued instructions from the select warps it waits for
      if (ARBOR_EVICT_SLEEP_NS) mbar_wait_sleep(&full[sl], (k / kJobSlots) & 1, ARBOR_EVICT_SLEEP_NS);
      else mbar_wait(&full[sl], (k / kJobSlots) & 1);
      if (kTrace && a.trace && k > 0) w_full += clock64() - tw0;
      if (k == 0) EV_TRACE(2);
      const int cnt = mycount[sl];
      if (cnt < 0) break;
      k_jobs = k + 1;
      const int nm = (kExp && (a.exp & 1)) ? 0 : cnt;
      const int2 *jb = myjobs + sl * jcap;
      move_rows<kUw>(nm, [&](int i) { return jb[i].x; }, [&](int i) { return jb[i].y; }, kp8, vp8,
                a.pos, rb, rpi, piece, sub);
      __syncwarp();
      if (lane == 0) mbar_arrive(&empty[sl]);
      if (kTrace && a.trace) mv_rows += cnt;
    }
    EV_TRACE(3);
    if (kTrace && a.trace && lane == 0) {   // diagnostics: SM id, jobs and rows this move warp handled
      unsigned smid;
      asm volatile("mov.u32 %0, %%smid;" : "=r"(smid));
      a.trace[(static_cast<int64_t>(blockIdx.x) * (2 * kPairsWs) + warp) * kTraceSlots + 7] =
          (static_cast<long long>(smid) << 40) | (static_cast<long long>(k_jobs) << 20) | mv_rows;
      a.trace[(static_cast<int64_t>(blockIdx.x) * (2 * kPairsWs) + warp) * kTraceSlots + 6] = w_full;   // cycles
    }
    return;
  }
  // -------------------------------------------------------------- select warp
  unsigned long long *key = reinterpret_cast<unsigned long long *>(sm + Ly.keys) + pid * cap;
  int32_t *holes = reinterpret_cast<int32_t *>(sm + Ly.lists) + pid * 2 * cap;
  int32_t *movers = holes + cap;
  float *Abuf = reinterpret_cast<float *>(sm + Ly.abuf) + pid * 2 * capA;
  int16_t *Pbuf = reinterpret_cast<int16_t *>(sm + Ly.pbuf) + pid * 2 * capP;
  int32_t *Gbuf = reinterpret_cast<int32_t *>(sm + Ly.gbuf) + pid * 3 * pcap;
  WorkEnt *Mbuf = reinterpret_cast<WorkEnt *>(sm + Ly.mbuf) + pid * 4;
  uint32_t *hist = hist_all[pid];
  const unsigned lt_mask = (1u << lane) - 1u;
  // pool row ids fit int32 (arbor_init checks L·NP·H·P < 2^31): 32-bit row math in the select
  // warp (one register and one add per use fewer than 64-bit offsets at the 64-register cap)
#ifndef ARBOR_EVICT_HOIST
#define ARBOR_EVICT_HOIST 1
#endif
#ifndef ARBOR_EVICT_ROW32
#define ARBOR_EVICT_ROW32 1
#endif
  using RowT = std::conditional_t<ARBOR_EVICT_ROW32 != 0, int, int64_t>;
  const RowT pstride = static_cast<RowT>(H) << lgP;
  constexpr unsigned long long kCand = 1ull << 63;
  // work items (changed node, row) are handed out dynamically — lane 0 draws the item of
  // pipeline step k + draw (ahead of the one being ranked) from a global counter — so
  // every pair finishes within about one item of the others (a static round robin left a
  // ~40 µs spread of finishing times on C2, profiles/evict_trace.py)
  // The draw for step k + draw is issued at the top of step k and stored at its end (its latency
  // hides behind the ranking).
  int *iring = reinterpret_cast<int *>(sm + Ly.iring) + pid * 4;
  int *wring = iring + 4 * kPairsWs;     // work entry of each slot's item (item / R, once)
  auto item_of = [&](int k) { return iring[k & 3]; };
  const WorkEnt *swl = reinterpret_cast<const WorkEnt *>(sm + Ly.swl);
  // work entry of pipeline step k: the shared-memory work list, or the cp.async'ed copy
  auto meta = [&](int k) -> const WorkEnt & {
    return Ly.wl_n ? swl[wring[k & 3]] : Mbuf[k & 3];
  };
  auto row_base = [&](int it, int w) -> RowT {
    const int r = it - w * a.R;
    const int l = r / H, h = r - l * H;
    return (static_cast<RowT>(l) * a.NP * H + h) << lgP;
  };
  // pipeline stages (each lane issues its share; completion via cp.async.wait_all + __syncwarp)
  auto issue_meta = [&](int k) {
    const int it = item_of(k);
    if (Ly.wl_n || it >= items || lane >= 2) return;
    const int w = wring[k & 3];
    cp_async16ca(reinterpret_cast<char *>(&Mbuf[k & 3]) + lane * 16,
                 reinterpret_cast<const char *>(&wl[w]) + lane * 16);
  };
  // page list of the valid slots: from the live page holding slot soff (Gbuf[0]); valid slot
  // s sits at Gbuf-relative slot (soff mod P) + s
  auto issue_pages = [&](int k) {
    if (item_of(k) >= items) return;
    const WorkEnt &e = meta(k);
    const int f0 = e.so >> lgP;
    const int np = ((e.so + e.kc + Pm) >> lgP) - f0;
    const int32_t *pl = a.ptab + static_cast<int64_t>(e.node) * a.MPN + f0;
    int32_t *g = Gbuf + (k % 3) * pcap;
    for (int i = lane; i < np; i += 32) cp_async4(g + i, pl + i);
  };
  // pos tags (need the page list) and the A span (needs only the work entry); a full node
  // (k_cur = n) holds its positions in slot order (appends and rehydration write the
  // identity, only an eviction permutes slots and it lowers k_cur): no pos tags to load
  auto issue_pos = [&](int k) {
    const int it = item_of(k);
    if (it >= items) return;
    const WorkEnt &e = meta(k);
    if (e.kc == e.n && e.so == 0) return;
    const int32_t *g = Gbuf + (k % 3) * pcap;
    const RowT base = row_base(it, wring[k & 3]);
    int16_t *pb = Pbuf + (k & 1) * capP;
    const int sb = e.so & Pm;
    // Gbuf-relative slot pairs (c even; P even: same page) covering [sb, sb + k_cur)
    for (int c = (sb & ~1) + 2 * lane; c < sb + e.kc; c += 64)
      cp_async4(pb + c, a.pos + (base + static_cast<RowT>(g[c >> lgP]) * pstride + (c & Pm)));
  };
  // the A row of pipeline step k's item over its span (A is read by position)
  auto a_row = [&](int k) -> const float * {
    const WorkEnt &e = meta(k);
    const int r = item_of(k) - wring[k & 3] * a.R;
    return a.Ahat ? a.Ahat + e.span : a.A + static_cast<int64_t>(r) * a.max_tokens + e.span;
  };
  // 16-byte cp.async from the span's aligned start: float p of the span lands at ab[mis + p]
  // (an aligned 16-byte chunk that overlaps the row never leaves its allocation)
  auto issue_A = [&](int k) {
    const int it = item_of(k);
    if (it >= items) return;
    const WorkEnt &e = meta(k);
    const int tl = min(a.l_tail, e.n);
    if (e.ka > tl && a.select_mode == ARBOR_SELECT_HEAVY) {   // ranked by A: the non-tail span
      const uintptr_t ar = reinterpret_cast<uintptr_t>(a_row(k));
      const char *a0 = reinterpret_cast<const char *>(ar & ~uintptr_t(15));
      const int nch = (static_cast<int>((ar & 15) >> 2) + e.n - tl + 3) >> 2;
      float *ab = Abuf + (k & 1) * capA;
      for (int c = lane; c < nch; c += 32) cp_async16(ab + 4 * c, a0 + 16 * c);
    }
  };
  // items are drawn `draw` pipeline steps ahead: 4 with a global work list (its entries are
  // fetched three steps ahead), 3 with the shared-memory list (page lists two steps ahead are
  // the farthest look-ahead) — every item drawn but not yet ranked when the counter runs out
  // is tail work for its warp alone.  The first `draw` items of select warp w are
  // draw·w … draw·w + draw − 1 (no atomic storm at the start); the counter hands out the
  // rest, from draw·(select warps) on
#ifndef ARBOR_EVICT_DRAW_SMEM
#define ARBOR_EVICT_DRAW_SMEM 3
#endif
  const int draw = Ly.wl_n ? ARBOR_EVICT_DRAW_SMEM : 4;
  const int nsel = static_cast<int>(gridDim.x) * kPairsWs;
  const int gw = static_cast<int>(blockIdx.x) * kPairsWs + pid;
  if (lane == 0) {
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      iring[i] = i < draw ? draw * gw + i : items;
      wring[i] = (draw * gw + i) / a.R;
    }
  }
  __syncwarp();
  // prologue: work entries 0-2 (smem list: nothing to fetch) → page lists 0, 1 and A of item 0
  // → pos tags of item 0 (none for a full node)
  issue_meta(0);
  issue_meta(1);
  issue_meta(2);
  cp_async_commit();
  cp_async_wait_all();
  __syncwarp();
  issue_pages(0);
  issue_pages(1);
  issue_A(0);
  cp_async_commit();
  cp_async_wait_all();
  __syncwarp();
  issue_pos(0);
  cp_async_commit();
  int k = 0;
  long long w_empty = 0;
#ifdef ARBOR_EVICT_PHASES
  long long ph[6] = {0, 0, 0, 0, 0, 0};
  long long ph_t = clock64();
#endif
  for (;; ++k) {
    const int it = item_of(k);
    if (it >= items) break;          // the counter only grows: every later draw is past the end
    int nxt = 0;
    if (lane == 0) nxt = draw * nsel + atomicAdd(&a.ctrl->item_next, 1);   // step k + draw's item
    cp_async_wait_all();
    __syncwarp();
    PH_MARK(5);
    issue_pos(k + 1);
    issue_A(k + 1);
    issue_pages(k + 2);
    issue_meta(k + 3);
    cp_async_commit();
    PH_MARK(0);
    // ---- rank item k from shared memory
    const WorkEnt e = meta(k);
    const bool ident = e.kc == e.n && e.so == 0;
    const int sb = e.so & Pm;
    if (k == 0) EV_TRACE(6);         // item 0's data landed: ranking starts
    const int kc = e.kc, ka = e.ka, n = e.n;
    const int tl = min(a.l_tail, n);
    const int32_t *pgs = Gbuf + (k % 3) * pcap;
    const int16_t *pb = Pbuf + (k & 1) * capP;
    const float *ab = Abuf + (k & 1) * capA +
                      ((reinterpret_cast<uintptr_t>(a_row(k)) & 15) >> 2);
    const RowT base = row_base(it, wring[k & 3]);
    auto row = [&](int slot) -> RowT {
      const int c = sb + slot;
      return base + static_cast<RowT>(pgs[c >> lgP]) * pstride + (c & Pm);
    };
    const bool ranked = ka > tl;
    const int m = ka - tl;
    const int tail_from = n - (ranked ? tl : ka);   // keep positions ≥ tail_from outright
    int ncand = 0;
    uint32_t bmin = 0xffffffffu, bmax = 0u;
    unsigned sink_all = 1u, sink_any = 0u;
#if ARBOR_EVICT_HOIST
    // positions below nsk are global sinks (0 unless this is the root under HEAVY / SINKS_TAIL);
    // an invalid A (NaN, negative, inf) is latched once per item, not branched on per slot
    const int nsk = (e.node == 0 && a.select_mode != ARBOR_SELECT_TAIL) ? a.n_sinks : 0;
    unsigned bad = 0u;
#endif
#pragma unroll kSelUnroll
    for (int s0 = 0; s0 < kc; s0 += 32) {
      const int s = s0 + lane;
      unsigned long long kk = 0;
      if (s < kc) {
        const int p = ident ? s : pb[sb + s];
        kk = static_cast<unsigned>(p);
        if (ranked && p < tail_from) {
          // key = ⟨sink, A bits, position⟩ (oracle/select.rank_key): the global sinks — the
          // root's first n_sinks positions — rank above everything else
          // in HEAVY and SINKS_TAIL (bit 48), then the f32 bits of A (HEAVY; 0 for the
          // recency rules TAIL, SINKS_TAIL), then the position
#if ARBOR_EVICT_HOIST
          const unsigned sink = p < nsk ? 1u : 0u;
#else
          const unsigned sink =
              (e.node == 0 && p < a.n_sinks && a.select_mode != ARBOR_SELECT_TAIL) ? 1u : 0u;
#endif
          unsigned bits = 0u;
          if (a.select_mode == ARBOR_SELECT_HEAVY) {
            const float av = ab[p];
#if ARBOR_EVICT_HOIST
            bad |= static_cast<unsigned>(!(av >= 0.f) || isinf(av));
#else
            if (!(av >= 0.f) || isinf(av)) atomicOr(&a.ctrl->err, DERR_INVARIANT);
#endif
            bits = (av == 0.f) ? 0u : __float_as_uint(av);   // −0 → +0 (Q3)
          }
          kk = kCand | (static_cast<unsigned long long>(sink) << 48) |
               (static_cast<unsigned long long>(bits) << 16) | static_cast<unsigned>(p);
          bmin = min(bmin, bits);
          bmax = max(bmax, bits);
          sink_all &= sink;
          sink_any |= sink;
        }
        key[s] = kk;
      }
      ncand += __popc(__ballot_sync(0xffffffffu, (kk & kCand) != 0));
    }
#if ARBOR_EVICT_HOIST
    if (bad) atomicOr(&a.ctrl->err, DERR_INVARIANT);
#endif
    __syncwarp();
    PH_MARK(1);
    // threshold: keep a candidate iff (key & tmask) >= tkey (the top m unique keys)
    unsigned long long tkey = kCand, tmask = kCand;     // m ≥ ncand: all candidates
    if (ranked && m <= 0) {
      tkey = ~0ull; tmask = ~0ull;                      // none survives
    } else if (ranked && m < ncand && !(kExp && (a.exp & 2))) {
      // candidates share every key bit above `top` (bits of A above the highest bit where
      // min and max differ); the radix passes start there
      bmin = __reduce_min_sync(0xffffffffu, bmin);
      bmax = __reduce_max_sync(0xffffffffu, bmax);
      sink_all = __reduce_and_sync(0xffffffffu, sink_all);
      sink_any = __reduce_or_sync(0xffffffffu, sink_any);
      // the sink bit differs among the candidates: start at bit 48
      const int top = sink_all != sink_any ? 48
                      : bmin != bmax ? 16 + 31 - __clz(static_cast<int>(bmin ^ bmax)) : 15;
      unsigned long long prefix = kCand, pmask = kCand;
      int need = m, inb = ncand;   // the need-th largest of the inb keys matching prefix
      // 8-bit digit passes while more than kFinish keys share the prefix
      for (int shift = top - 7; shift > -8 && inb > kFinish && need < inb; shift -= 8) {
        const unsigned long long dmask = shift >= 0 ? 255ull << shift : 255ull >> -shift;
        reinterpret_cast<uint4 *>(hist)[2 * lane] = make_uint4(0u, 0u, 0u, 0u);
        reinterpret_cast<uint4 *>(hist)[2 * lane + 1] = make_uint4(0u, 0u, 0u, 0u);
        __syncwarp();
#pragma unroll kSelUnroll
        for (int s = lane; s < kc; s += 32) {
          const unsigned long long kk = key[s];
          if ((kk & pmask) == prefix) {
            const unsigned dg = shift >= 0 ? static_cast<unsigned>(kk >> shift) & 255u
                                           : static_cast<unsigned>(kk << -shift) & 255u;
            atomicAdd(&hist[dg], 1u);
          }
        }
        __syncwarp();
        // lane j scans digits 255 − 8j … 248 − 8j (descending): bins 8(31 − j) … 8(31 − j) + 7
        const uint4 h0 = reinterpret_cast<const uint4 *>(hist)[2 * (31 - lane)];
        const uint4 h1 = reinterpret_cast<const uint4 *>(hist)[2 * (31 - lane) + 1];
        const uint32_t cnt8[8] = {h1.w, h1.z, h1.y, h1.x, h0.w, h0.z, h0.y, h0.x};
        uint32_t loc = 0;
#pragma unroll
        for (int b = 0; b < 8; ++b) loc += cnt8[b];
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
        inb = static_cast<int>(inbin);
      }
      tkey = prefix;
      tmask = pmask;
      if (need < inb) {
        // finish (≤ kFinish keys left in the prefix's bin): gather them, one per lane, and
        // take the one with exactly need − 1 larger keys (keys are unique) — replaces the
        // remaining digit passes; `holes` is scratch here (written only below)
        unsigned long long *bin = reinterpret_cast<unsigned long long *>(holes);
        int c = 0;
    #pragma unroll kSelUnroll
    for (int s0 = 0; s0 < kc; s0 += 32) {
          const int s = s0 + lane;
          const unsigned long long kk = s < kc ? key[s] : 0ull;
          const bool in = s < kc && (kk & pmask) == prefix;
          const unsigned bb = __ballot_sync(0xffffffffu, in);
          if (in) bin[c + __popc(bb & lt_mask)] = kk;
          c += __popc(bb);
        }
        __syncwarp();
        const unsigned long long mk = lane < inb ? bin[lane] : 0ull;
        int gt = 0;
        for (int j = 0; j < inb; ++j) gt += __shfl_sync(0xffffffffu, mk, j) > mk ? 1 : 0;
        const unsigned hit = __ballot_sync(0xffffffffu, lane < inb && gt == need - 1);
        if (hit) {                        // else non-unique keys (corrupted state): latched below
          tkey = __shfl_sync(0xffffffffu, mk, __ffs(hit) - 1);
          tmask = ~0ull;
        }
        __syncwarp();
      }
    }
    PH_MARK(2);
    // keep flags → holes (dropped slots of the window [k_cur − k_app, k_cur)) and movers
    // (kept slots before it), ascending
    const int w0 = kc - ka;
    int nh = 0, nm = 0;
#pragma unroll kUnrollLists
    for (int s0 = 0; s0 < kc; s0 += 32) {
      const int s = s0 + lane;
      int keep = 0;
      if (s < kc) {
        const unsigned long long kk = key[s];
        const int p = static_cast<int>(kk & 0xffffu);
        // branch-free (the short-circuit form compiled to a divergent branch per slot)
        keep = static_cast<int>(p >= tail_from) |
               (static_cast<int>(ranked) & static_cast<int>(kk >> 63) &
                static_cast<int>((kk & tmask) >= tkey));
      }
      const int hole = s >= w0 && s < kc && !keep;
      const int mv = s < w0 && keep;
      const unsigned hb = __ballot_sync(0xffffffffu, hole);
      const unsigned mb = __ballot_sync(0xffffffffu, mv);
      if (hole) holes[nh + __popc(hb & lt_mask)] = s;
      if (mv) movers[nm + __popc(mb & lt_mask)] = s;
      nh += __popc(hb);
      nm += __popc(mb);
    }
    __syncwarp();
    // holes and movers pair up exactly when the kept keys are unique (they are for a
    // consistent state: one pos tag per position); otherwise latch the error and move only the
    // pairs that exist, so a corrupted state can never produce out-of-range rows
    if (nh != nm && lane == 0 && !(kExp && a.exp)) atomicOr(&a.ctrl->err, DERR_STATE);
    nm = nm < nh ? nm : nh;
    PH_MARK(3);
    // hand the job to the move warp
    const int sl = k & (kJobSlots - 1);
    const long long tw0 = (kTrace && a.trace) ? clock64() : 0;
    if (ARBOR_EVICT_SLEEP_NS) mbar_wait_sleep(&empty[sl], ((k / kJobSlots) & 1) ^ 1, ARBOR_EVICT_SLEEP_NS);
    else mbar_wait(&empty[sl], ((k / kJobSlots) & 1) ^ 1);
    if (kTrace && a.trace) w_empty += clock64() - tw0;
    int2 *jb = myjobs + sl * jcap;
    for (int i = lane; i < nm; i += 32)
      jb[i] = make_int2(static_cast<int>(row(movers[i])), static_cast<int>(row(holes[i])));
    if (lane == 0) {
      mycount[sl] = nm;
      iring[(k + draw) & 3] = nxt;   // step k + draw (read after the next step's __syncwarp)
      wring[(k + draw) & 3] = nxt / a.R;
    }
    __syncwarp();
    if (lane == 0) mbar_arrive(&full[sl]);
    if (k == 0) EV_TRACE(2);
    PH_MARK(4);
  }
#ifdef ARBOR_EVICT_PHASES
  if (kTrace && a.trace && lane == 0)
    for (int i = 0; i < 6; ++i)
      a.trace[(static_cast<int64_t>(blockIdx.x) * (2 * kPairsWs) + warp) * kTraceSlots + 8 + i] = ph[i];
  if (kTrace && a.trace && lane == 0)
    a.trace[(static_cast<int64_t>(blockIdx.x) * (2 * kPairsWs) + warp) * kTraceSlots + 14] = k;
#endif
  cp_async_wait_all();               // prefetches past the end (none were issued, but be tidy)
  // end marker for the move warp
  {
    const int sl = k & (kJobSlots - 1);
    mbar_wait(&empty[sl], ((k / kJobSlots) & 1) ^ 1);
    if (lane == 0) {
      mycount[sl] = -1;
      mbar_arrive(&full[sl]);
    }
  }
  // the last select warp past the end resets the counters for the next launch (every draw
  // of this launch has happened by then)
  if (lane == 0) {
    __threadfence();
    if (atomicAdd(&a.ctrl->item_done, 1) == nsel - 1) {
      a.ctrl->item_next = 0;
      a.ctrl->item_done = 0;
    }
  }
  EV_TRACE(3);
  if (kTrace && a.trace && lane == 0)   // diagnostics: cycles this select warp waited for a free job slot
    a.trace[(static_cast<int64_t>(blockIdx.x) * (2 * kPairsWs) + warp) * kTraceSlots + 7] = w_empty;
}

}  // namespace

// Â[t] = Σ_{(l,h) ∈ slice, ascending} A[l][h][t]: fp64 accumulation of the f32 values, one
// f32 rounding (the oracle's definition, bit for bit); grid-stride over positions
__global__ void ahat_kernel(const float *__restrict__ A, int L, int H, int64_t max_tokens,
                            SliceView sv, float *__restrict__ out) {
  for (int64_t t = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; t < max_tokens;
       t += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    double acc = 0.0;
    for (int l = 0; l < L; ++l)
      for (int h = 0; h < H; ++h)
        if (sv.has(l, h)) acc = __dadd_rn(acc, static_cast<double>(A[(static_cast<int64_t>(l) * H + h) * max_tokens + t]));
    out[t] = __double2float_rn(acc);
  }
}

long long *g_evict_trace = nullptr;
size_t g_evict_trace_n = 0;

void launch_ahat(arbor_ctx *c) {
  const int grid = static_cast<int>(std::min<int64_t>((c->max_tokens + 255) / 256, 4 * c->num_sms));
  ahat_kernel<<<grid, 256, 0, c->ms>>>(c->cfg.score, c->L, c->H, c->max_tokens, slice_view(c),
                                       c->d.ahat);
  ARBOR_LAUNCHED(c);
}

void launch_evict(arbor_ctx *c, int N, const int32_t *k_target, int max_n, bool gated) {
  CompactArgs a{};
  a.gate = gated ? &c->d.ctrl->gate : nullptr;
  a.R = c->L * c->H;
  a.H = c->H;
  a.P = c->P;
  a.D = c->D;
  a.NP = c->NP;
  a.MPN = c->max_pages_node;
  a.l_tail = c->prm.l_tail;
  a.max_tokens = c->max_tokens;
  a.work = c->d.work;
  a.N = N;
  a.MN = c->max_nodes;
  a.k_target = k_target;
  a.n = c->d.n;
  a.pinned = c->d.pinned;
  a.span = c->d.span;
  a.kcur = c->d.kcur;
  a.soff = c->d.soff;
  a.npages = c->d.npages;
  a.free_stack = c->d.free_stack;
  a.A = c->cfg.score;
  a.Ahat = c->prm.select_shared ? c->d.ahat : nullptr;
  a.ctrl_ro = c->d.ctrl;
  a.ctrl = c->d.ctrl;
  a.ptab = c->d.ptab;
  a.kpool = c->cfg.k_pool;
  a.vpool = c->cfg.v_pool;
  a.pos = c->cfg.pos_pool;
  a.esize = c->esize;
  a.cap = max_n < 1 ? 1 : max_n;
  a.lgP = __builtin_ctz(static_cast<unsigned>(c->P));
  a.select_mode = c->prm.select_mode;
  a.n_sinks = c->prm.n_sinks;
  static const int exp_flags = [] {
    const char *e = getenv("ARBOR_EVICT_EXP");
    return e ? atoi(e) : 0;
  }();
  a.exp = exp_flags;
  a.trace = nullptr;
  a.wl_smem = N <= kSmemWorkNodes ? N : 0;
  static long long *trace = nullptr;
  static size_t trace_n = 0;
  if (getenv("ARBOR_EVICT_TRACE")) {
    const size_t need = static_cast<size_t>(c->num_sms) * kEvictCtasPerSm * 2 * kPairsWs * kTraceSlots;
    if (need > trace_n) {
      if (trace) cudaFree(trace);
      cudaMalloc(&trace, need * sizeof(long long));
      trace_n = need;
    }
    cudaMemsetAsync(trace, 0, trace_n * sizeof(long long), c->ms);
    a.trace = trace;
    g_evict_trace = trace;
    g_evict_trace_n = trace_n;
  }
  // the fixed-layout instantiation for the common shape: nodes of ≤ 128 slots, 16-slot pages,
  // 8 KV heads (the Llama-3.1-8B / Qwen2.5-32B shapes of C2-C5)
#ifndef ARBOR_EVICT_FIXED
#define ARBOR_EVICT_FIXED 1
#endif
  const bool fixed = ARBOR_EVICT_FIXED && a.cap <= 128 && a.lgP == 4 && a.H == 8;
  if (fixed) a.cap = 128;
  const WsLayout ly(a.cap, a.lgP, a.wl_smem);
  const int inst = fixed ? 1 : 0;
  auto kfn = fixed ? select_move_ws_kernel<128, 4, 8> : select_move_ws_kernel<0, 0, 0>;
  // both instantiations are loaded on the first call (lazy loading would otherwise load the
  // runtime-layout one the first time a node above 128 slots is evicted: a millisecond-scale
  // stall in the middle of a run, e.g. C3's e2e)
  static const bool loaded = [] {
    cudaFuncAttributes fa;
    cudaFuncGetAttributes(&fa, select_move_ws_kernel<128, 4, 8>);
    cudaFuncGetAttributes(&fa, select_move_ws_kernel<0, 0, 0>);
    return true;
  }();
  (void)loaded;
  // occupancy / smem attribute cached per instantiation and layout (host-side cost stays off
  // the launch path)
  static size_t attr_smem[2] = {0, 0};
  static size_t cached_total[2] = {0, 0};
  static int cached_grid[2] = {0, 0};
  if (ly.total > attr_smem[inst]) {
    const size_t want = ly.total < 48 * 1024 ? 48 * 1024 : ly.total;
    cudaFuncSetAttribute(kfn, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(want));
    attr_smem[inst] = want;
  }
  if (ly.total != cached_total[inst]) {
    int sms = 148, per = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, kfn, kPairsWs * 64, ly.total);
    cached_grid[inst] = sms * std::min(std::max(per, 1), kEvictCtasPerSm);
    cached_total[inst] = ly.total;
  }
  stage_begin(c, ARBOR_ST_SELECT_COMPACT, c->ms);
  launch_pdl(kfn, dim3(cached_grid[inst]), dim3(kPairsWs * 64), ly.total, c->ms, a);
  ARBOR_LAUNCHED(c);
  stage_end(c, ARBOR_ST_SELECT_COMPACT, c->ms);
}

}  // namespace arbor

// debug only (not part of include/arbor.h): the last ARBOR_EVICT_TRACE timeline
// ([cta][16 warps][8] globaltimer ns; warps 0-7 select, 8-15 move) and its grid size
extern "C" int arbor_debug_evict_trace(long long *host, long long count) {
  if (!arbor::g_evict_trace || count < 0 || static_cast<size_t>(count) > arbor::g_evict_trace_n) return -1;
  cudaDeviceSynchronize();
  return cudaMemcpy(host, arbor::g_evict_trace, sizeof(long long) * count, cudaMemcpyDeviceToHost) == cudaSuccess ? 0 : -2;
}
