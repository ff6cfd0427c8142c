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
//  * select_compact (persistent grid, one WARP per (node, row) work item, no block
//    barriers): gathers the pos tags and A keys of the non-tail kept slots, finds the m-th
//    largest unique 48-bit key ⟨A bits, pos⟩ by a warp radix select (8-bit digits, per-warp
//    256-bin smem histogram, warp scan) — exact top-m membership in O(c) — warp-scans the keep
//    mask (ballot/popc) into new slot indices, then moves K, V and pos rows in ascending
//    slot order, in place: a kept row's new slot is never after its old one, and each chunk
//    of rows is fully read (16-byte coalesced loads, 8 rows in flight per warp) before any
//    of it is written.
#include <cub/block/block_scan.cuh>

#include "common.cuh"

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
    const int32_t *pl = a.ptab + static_cast<int64_t>(j) * a.MPN;
    for (int t = 0; t < fr[i]; ++t) a.free_stack[top + free_off + t] = pl[newp[i] + t];
    free_off += fr[i];
    a.npages[j] = newp[i];
    a.kcur[j] = kapp[i];
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    a.ctrl->free_top = top + tot_free;
    a.ctrl->work_count = tot_work;
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
  int esize;
  int cap;          // max n over evicted nodes (smem capacity, slots)
  int lgP;          // log2(page size)
};

__device__ __forceinline__ int64_t row_of(const CompactArgs &a, const int32_t *pl, int l, int h,
                                          int slot) {
  return ((static_cast<int64_t>(l) * a.NP + pl[slot / a.P]) * a.H + h) * a.P + (slot % a.P);
}

constexpr int kWarps = 8;     // warps per CTA; one warp owns one (node, row) work item
constexpr int kUnroll = 4;    // row-chunks in flight per lane during the move

// Warp-per-item select + compact.  smem per warp: key[cap] (u64), the move list[cap]
// (u32: src slot | dst slot << 16) and the node's page list[cap / P + 1].
__global__ void __launch_bounds__(kWarps * 32, 4)
select_compact_kernel(CompactArgs a) {
  extern __shared__ __align__(16) unsigned char sm[];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int cap = a.cap;
  const int lgP = a.lgP, Pm = (1 << lgP) - 1;
  const int pcap = (cap >> lgP) + 1;
  unsigned long long *key = reinterpret_cast<unsigned long long *>(sm) + warp * cap;
  uint32_t *mlist = reinterpret_cast<uint32_t *>(reinterpret_cast<unsigned long long *>(sm) +
                                                 kWarps * cap) + warp * cap;
  int32_t *pgs = reinterpret_cast<int32_t *>(reinterpret_cast<uint32_t *>(
                     reinterpret_cast<unsigned long long *>(sm) + kWarps * cap) + kWarps * cap) +
                 warp * pcap;
  __shared__ uint32_t hist_all[kWarps][256];
  uint32_t *hist = hist_all[warp];
  const int items = a.ctrl_ro->work_count * a.R;
  const int rb = a.D * a.esize;          // row bytes
  const int cpr = rb >> 4;               // 16-byte pieces per row (≤ 32)
  const int rpi = 32 / cpr;              // rows per warp instruction
  const int my_piece = lane % cpr, my_row = lane / cpr;
  const unsigned lt_mask = (1u << lane) - 1u;
  char *kp8 = static_cast<char *>(a.kpool);
  char *vp8 = static_cast<char *>(a.vpool);
  const int64_t pstride = static_cast<int64_t>(a.H) << lgP;   // rows between consecutive pages
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
    // 1. candidates: when k_app > |𝒯| the tail (the last |𝒯| slots, all present) is kept and
    //    the non-tail slots 0..nc-1 compete by key; otherwise the last k_app slots are kept
    //    (Alg. 1) and no key is needed.
    const bool ranked = ka > tl;
    const int nc = ranked ? kc - tl : 0;
    const int m = ka - tl;
    // threshold: keep a candidate iff (key & tmask) >= tkey — the top m keys (unique)
    unsigned long long tkey = ~0ull, tmask = ~0ull;
    if (ranked) {
      const float *Arow =
          a.A + (static_cast<int64_t>(l) * a.H + h) * a.max_tokens + a.span[node];
      for (int s = lane; s < nc; s += 32) {
        const int p = a.pos[row(s)];
        const float av = Arow[p];
        if (!(av >= 0.f) || isinf(av)) atomicOr(&a.ctrl->err, DERR_INVARIANT);
        const unsigned bits = (av == 0.f) ? 0u : __float_as_uint(av);   // −0 → +0 (Q3)
        key[s] = (static_cast<unsigned long long>(bits) << 16) | static_cast<unsigned>(p);
      }
      __syncwarp();
      if (m <= 0) {
        tkey = ~0ull;                      // no heavy hitter survives
      } else if (m >= nc) {
        tkey = 0; tmask = 0;               // every candidate survives
      } else {
        // warp radix select of the m-th largest 48-bit key, 8-bit digits MSB first
        unsigned long long prefix = 0, pmask = 0;
        int need = m;
        for (int shift = 40; shift >= 0; shift -= 8) {
#pragma unroll
          for (int b = 0; b < 8; ++b) hist[lane * 8 + b] = 0;
          __syncwarp();
          for (int s = lane; s < nc; s += 32) {
            const unsigned long long k = key[s];
            if ((k & pmask) == prefix) atomicAdd(&hist[(k >> shift) & 255u], 1u);
          }
          __syncwarp();
          // lane owns digits 255-8*lane … 248-8*lane (descending); counts from the top
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
          const bool mine = before < static_cast<uint32_t>(need) &&
                            static_cast<uint32_t>(need) <= incl;
          int dsel = 0;
          uint32_t above = 0, inbin = 0;
          if (mine) {
            uint32_t acc = before;
#pragma unroll
            for (int b = 0; b < 8; ++b) {
              if (acc < static_cast<uint32_t>(need) && static_cast<uint32_t>(need) <= acc + c[b] &&
                  inbin == 0) {
                dsel = 255 - lane * 8 - b;
                above = acc;
                inbin = c[b];
              }
              acc += c[b];
            }
          }
          const unsigned who = __ballot_sync(0xffffffffu, mine);
          const int src = __ffs(who) - 1;
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
    }
    // 2. keep decision, warp scan of the keep mask in slot order → new slot, move list
    int carry = 0, nmoves = 0;
    for (int b0 = 0; b0 < kc; b0 += 32) {
      const int s = b0 + lane;
      int keep = 0;
      if (s < kc) {
        if (!ranked) keep = s >= kc - ka;
        else if (s >= nc) keep = 1;                                  // tail 𝒯_i
        else keep = (key[s] & tmask) >= tkey;                        // Top-m_i by A_i(t)
      }
      const unsigned kb = __ballot_sync(0xffffffffu, keep);
      const int ns = carry + __popc(kb & lt_mask);
      carry += __popc(kb);
      const int mv = keep && ns != s;
      const unsigned mb = __ballot_sync(0xffffffffu, mv);
      if (mv) mlist[nmoves + __popc(mb & lt_mask)] = static_cast<uint32_t>(s) |
                                                      (static_cast<uint32_t>(ns) << 16);
      nmoves += __popc(mb);
    }
    __syncwarp();
    // 3. in-place stable gather: each chunk of rows is read completely into registers
    //    before any of it is written (a kept row never moves to a later slot)
    const int chunk_rows = rpi * kUnroll;
    for (int c0 = 0; c0 < nmoves; c0 += chunk_rows) {
      uint4 bk[kUnroll], bv[kUnroll];
      int16_t ptag[kUnroll];
#pragma unroll
      for (int u = 0; u < kUnroll; ++u) {
        const int rr = c0 + u * rpi + my_row;
        if (rr < nmoves) {
          const int64_t srow = row(static_cast<int>(mlist[rr] & 0xffffu));
          const int64_t off = srow * rb + my_piece * 16;
          bk[u] = *reinterpret_cast<const uint4 *>(kp8 + off);
          bv[u] = *reinterpret_cast<const uint4 *>(vp8 + off);
          if (my_piece == 0) ptag[u] = a.pos[srow];
        }
      }
      __syncwarp();
#pragma unroll
      for (int u = 0; u < kUnroll; ++u) {
        const int rr = c0 + u * rpi + my_row;
        if (rr < nmoves) {
          const int64_t drow = row(static_cast<int>(mlist[rr] >> 16));
          const int64_t off = drow * rb + my_piece * 16;
          *reinterpret_cast<uint4 *>(kp8 + off) = bk[u];
          *reinterpret_cast<uint4 *>(vp8 + off) = bv[u];
          if (my_piece == 0) a.pos[drow] = ptag[u];
        }
      }
      __syncwarp();
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
  a.esize = c->esize;
  const int cap = max_n < 1 ? 1 : max_n;
  a.cap = cap;
  a.lgP = __builtin_ctz(static_cast<unsigned>(c->P));
  const size_t smem = (static_cast<size_t>(cap) * (8 + 4) + ((cap >> a.lgP) + 1) * 4) * kWarps;
  static int attr_smem = 0;
  if (static_cast<int>(smem) > attr_smem) {
    cudaFuncSetAttribute(select_compact_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         static_cast<int>(smem) < 48 * 1024 ? 48 * 1024 : static_cast<int>(smem));
    attr_smem = static_cast<int>(smem) < 48 * 1024 ? 48 * 1024 : static_cast<int>(smem);
  }
  int blocks_per_sm = 0;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&blocks_per_sm, select_compact_kernel,
                                                kWarps * 32, smem);
  int sms = 148;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  const int grid = sms * (blocks_per_sm > 0 ? blocks_per_sm : 1);
  stage_begin(c, ARBOR_ST_SELECT_COMPACT, c->ms);
  select_compact_kernel<<<grid, kWarps * 32, smem, c->ms>>>(a);
  ARBOR_LAUNCHED(c);
  stage_end(c, ARBOR_ST_SELECT_COMPACT, c->ms);
}

}  // namespace arbor
