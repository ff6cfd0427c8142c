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
//  * select_compact (persistent grid, one CTA per (node, row) work item): gathers the pos
//    tags and A keys of the kept slots, ranks the non-tail candidates (unique keys → exact
//    rank = top-m membership), block-scans the keep mask into new slot indices, then moves
//    K, V and pos rows in ascending slot order, in place: a kept row's new slot is never
//    after its old one, and each 32-row chunk is fully read (into registers, 16-byte
//    coalesced loads) before any of it is written.
#include <cub/block/block_scan.cuh>

#include "common.cuh"

namespace arbor {
namespace {

constexpr int kPlanThreads = 1024;
constexpr int kCompactThreads = 128;

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
};

__device__ __forceinline__ int64_t row_of(const CompactArgs &a, const int32_t *pl, int l, int h,
                                          int slot) {
  return ((static_cast<int64_t>(l) * a.NP + pl[slot / a.P]) * a.H + h) * a.P + (slot % a.P);
}

// smem: key (u64) [max_n], pos (i32) [max_n], keep/new slot (i32) [max_n], moves (i32) [max_n]
__global__ void __launch_bounds__(kCompactThreads)
select_compact_kernel(CompactArgs a) {
  extern __shared__ __align__(16) unsigned char sm[];
  using Scan = cub::BlockScan<int, kCompactThreads>;
  __shared__ typename Scan::TempStorage tmp;
  __shared__ int s_moves, s_carry;
  const int items = a.ctrl_ro->work_count * a.R;
  const int cap = a.cap;
  unsigned long long *key = reinterpret_cast<unsigned long long *>(sm);
  int *pos = reinterpret_cast<int *>(key + cap);
  int *nslot = pos + cap;
  int *mv_src = nslot + cap;
  const int rb = a.D * a.esize;          // row bytes
  const int cpr = rb / 16;               // 16-byte chunks per row
  for (int it = blockIdx.x; it < items; it += gridDim.x) {
    const int w = it / a.R, r = it - w * a.R;
    const int l = r / a.H, h = r - l * a.H;
    const int node = a.work_node[w];
    const int kc = a.work_old[w], ka = a.work_new[w];
    const int n = a.n[node];
    const int tl = min(a.l_tail, n);
    const int32_t *pl = a.ptab + static_cast<int64_t>(node) * a.MPN;
    const float *Arow = a.A + (static_cast<int64_t>(l) * a.H + h) * a.max_tokens + a.span[node];
    // 1. gather pos tags and keys of the kept slots
    for (int s = threadIdx.x; s < kc; s += blockDim.x) {
      const int p = a.pos[row_of(a, pl, l, h, s)];
      pos[s] = p;
      const float av = Arow[p];
      if (!(av >= 0.f) || isinf(av)) atomicOr(&a.ctrl->err, DERR_INVARIANT);
      const unsigned bits = (av == 0.f) ? 0u : __float_as_uint(av);   // −0 → +0 (Q3)
      key[s] = (static_cast<unsigned long long>(bits) << 32) | static_cast<unsigned>(p);
    }
    __syncthreads();
    // 2. keep decision: tail, or top-(ka − tl) non-tail by key (exact rank, keys are unique)
    const int m = ka - tl;
    for (int s = threadIdx.x; s < kc; s += blockDim.x) {
      int keep;
      if (ka <= tl) {
        keep = pos[s] >= n - ka;                       // Alg. 1
      } else if (pos[s] >= n - tl) {
        keep = 1;                                      // tail 𝒯_i
      } else {
        const unsigned long long ks = key[s];
        int rank = 0;
        for (int i = 0; i < kc; ++i)
          rank += (pos[i] < n - tl) && (key[i] > ks);
        keep = rank < m;                               // Top-m_i by A_i(t)
      }
      nslot[s] = keep;
    }
    __syncthreads();
    // 3. block scan of the keep mask in slot order → new slot; collect moving rows
    if (threadIdx.x == 0) { s_carry = 0; s_moves = 0; }
    __syncthreads();
    for (int base = 0; base < kc; base += blockDim.x) {
      const int s = base + threadIdx.x;
      const int kp = (s < kc) ? nslot[s] : 0;
      int ex;
      Scan(tmp).ExclusiveSum(kp, ex);
      const int carry = s_carry;
      __syncthreads();
      if (s < kc) nslot[s] = kp ? (carry + ex) : -1;
      if (threadIdx.x == blockDim.x - 1) s_carry = carry + ex + kp;
      __syncthreads();
    }
    // moving rows (new slot != old slot), in ascending slot order
    for (int base = 0; base < kc; base += blockDim.x) {
      const int s = base + threadIdx.x;
      const int mvf = (s < kc && nslot[s] >= 0 && nslot[s] != s) ? 1 : 0;
      int ex;
      Scan(tmp).ExclusiveSum(mvf, ex);
      const int carry = s_moves;
      __syncthreads();
      if (mvf) mv_src[carry + ex] = s;
      if (threadIdx.x == blockDim.x - 1) s_moves = carry + ex + mvf;
      __syncthreads();
    }
    const int moves = s_moves;
    // 4. in-place stable gather, chunks of 32 rows: read all, sync, write all
    constexpr int kChunkRows = 32;
    char *kp8 = static_cast<char *>(a.kpool);
    char *vp8 = static_cast<char *>(a.vpool);
    for (int c0 = 0; c0 < moves; c0 += kChunkRows) {
      const int nr = min(kChunkRows, moves - c0);
      const int pieces = nr * cpr;   // per tensor
      uint4 bufk[8], bufv[8];       // kChunkRows * cpr / threads ≤ 32*16/128 = 4 (bf16, d=128)
      int npc = 0;
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        const int pc = threadIdx.x + u * kCompactThreads;
        if (pc < pieces) {
          const int rr = pc / cpr, cc = pc - rr * cpr;
          const int src = mv_src[c0 + rr];
          const int64_t off = row_of(a, pl, l, h, src) * rb + cc * 16;
          bufk[u] = *reinterpret_cast<const uint4 *>(kp8 + off);
          bufv[u] = *reinterpret_cast<const uint4 *>(vp8 + off);
          npc = u + 1;
        }
      }
      __syncthreads();
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        const int pc = threadIdx.x + u * kCompactThreads;
        if (u < npc && pc < pieces) {
          const int rr = pc / cpr, cc = pc - rr * cpr;
          const int src = mv_src[c0 + rr];
          const int64_t off = row_of(a, pl, l, h, nslot[src]) * rb + cc * 16;
          *reinterpret_cast<uint4 *>(kp8 + off) = bufk[u];
          *reinterpret_cast<uint4 *>(vp8 + off) = bufv[u];
        }
      }
      for (int rr = threadIdx.x; rr < nr; rr += blockDim.x) {
        const int src = mv_src[c0 + rr];
        a.pos[row_of(a, pl, l, h, nslot[src])] = static_cast<int16_t>(pos[src]);
      }
      __syncthreads();
    }
    __syncthreads();
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
  const size_t smem = static_cast<size_t>(cap) * (8 + 4 + 4 + 4);
  static int attr_smem = 0;
  if (static_cast<int>(smem) > attr_smem) {
    cudaFuncSetAttribute(select_compact_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         static_cast<int>(smem) < 48 * 1024 ? 48 * 1024 : static_cast<int>(smem));
    attr_smem = static_cast<int>(smem) < 48 * 1024 ? 48 * 1024 : static_cast<int>(smem);
  }
  int blocks_per_sm = 0;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&blocks_per_sm, select_compact_kernel,
                                                kCompactThreads, smem);
  int sms = 148;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  const int grid = sms * (blocks_per_sm > 0 ? blocks_per_sm : 1);
  stage_begin(c, ARBOR_ST_SELECT_COMPACT, c->ms);
  select_compact_kernel<<<grid, kCompactThreads, smem, c->ms>>>(a);
  ARBOR_LAUNCHED(c);
  stage_end(c, ARBOR_ST_SELECT_COMPACT, c->ms);
}

}  // namespace arbor
