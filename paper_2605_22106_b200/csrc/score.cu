// score.cu — §8(a) a2 (accumulated attention), a3 (node mass + MSVE).
//
// a2 (§4 Execution (iii)): A_i(t) = Σ_{u>b_i} Σ_l Σ_h Attn_{u→t}.  Per
// decode step and active leaf b: p_t = exp(q·k_t/√d − LSE_{b,l,g}) over the visible slots
// of Path(ℓ_b), A[l][h][a_j + pos_t] += Σ_{g∈group(h)} p_t — computed from the logits the
// attention kernel already produced ("from attention weights already materialized during
// decoding"), without re-reading K.
//
// a3 (Q4/Q5/Q29): m_{l,h,i} = Σ_{t∈span_i} A[l][h][t] accumulated in fp64,
// Q = round-half-even(m · 2^24) as int64, Mass_i = Σ_rows Q (exact int64 sums: order- and
// world-size-independent).  A changes only at the visible tokens of a score call, so each
// rank caches its per-node partial Q sum and recomputes it for the visible closed nodes only; a_i = clamp((Mass_i − Mclose_i) 2^-24 / (Nq_i L Hq), 0, 1);
// s_i = clip(σ(θ0 + θ_v v_i + θ_u u_i + θ_a a_i), 0, 1) in fp64, rounded to f32.
#include "tile.cuh"

namespace arbor {
namespace {

constexpr float kLog2e = 1.4426950408889634f;

// Arguments of the score pass (a2) over the attention kernel's logits (zbuf).
struct ApplyArgs {
  PlanView pv;
  PoolView g;
  const int16_t *pos;
  const int32_t *ptab, *kcur, *soff;
  const int64_t *span;
  const float *zbuf, *lse;
  float *A;
  Ctrl *ctrl;
  int Lc, Hq, G;
};

// Node mass in two launches: one CTA per (listed node, layer) — warps over the layer's KV
// heads, each warp sums one row of A over the node's span in fp64 (lanes strided, xor tree:
// fixed order) and quantises Q = round-half-even(m · 2^24); the CTA's int64 sum goes to
// scratch[node_idx][layer]; a finalize kernel adds the layers (exact integer sums) and
// writes out[node * out_stride].
constexpr int kMassThreads = 256;
__global__ void __launch_bounds__(kMassThreads)
node_mass_kernel(const int32_t *__restrict__ nodes, const int32_t *__restrict__ nlen,
                 const int64_t *__restrict__ span, const float *__restrict__ A, int L, int H,
                 int64_t max_tokens, int64_t *__restrict__ scratch, SliceView sv) {
  const int node = nodes[blockIdx.x];
  const int l = blockIdx.y;
  const int n = nlen[node];
  const int64_t a0 = span[node];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  constexpr int kW = kMassThreads / 32;
  __shared__ long long red[kW];
  long long qsum = 0;
  for (int h = warp; h < H; h += kW) {
    if (!sv.has(l, h)) continue;                  // thin slice (Q6)
    const float *row = A + (static_cast<int64_t>(l) * H + h) * max_tokens + a0;
    double m = 0.0;
    for (int t = lane; t < n; t += 32) m += static_cast<double>(row[t]);
#pragma unroll
    for (int o = 16; o; o >>= 1) m += __shfl_xor_sync(0xffffffffu, m, o);
    qsum += __double2ll_rn(m * 16777216.0);   // round-half-even(m · 2^24), all lanes agree
  }
  if (lane == 0) red[warp] = qsum;
  __syncthreads();
  if (threadIdx.x == 0) {
    long long tot = 0;
    for (int w = 0; w < kW; ++w) tot += red[w];
    scratch[static_cast<int64_t>(blockIdx.x) * L + l] = tot;
  }
}

__global__ void node_mass_finalize(const int32_t *__restrict__ nodes, int count, int L,
                                   const int64_t *__restrict__ scratch, int64_t *__restrict__ out,
                                   int out_stride) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= count) return;
  long long tot = 0;
  for (int l = 0; l < L; ++l) tot += scratch[static_cast<int64_t>(i) * L + l];
  out[static_cast<int64_t>(nodes[i]) * out_stride] = tot;
}

struct MsveArgs {
  int N;
  const uint8_t *open;
  const float *v, *u;
  const int64_t *mass2;   // [0,N): Mass, [N,2N): Mclose (all-reduced)
  const int64_t *nq;
  double norm;            // L_global · Hq_global
  double th0, thv, thu, tha;
  float *a_out, *s_state, *s_out;
};

__global__ void msve_kernel(MsveArgs m) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= m.N) return;
  float s = 0.5f, af = 0.f;
  if (!m.open[i]) {
    double a = 0.0;
    const long long nq = m.nq[i];
    if (nq > 0) {
      const double num = static_cast<double>(m.mass2[i] - m.mass2[m.N + i]) * (1.0 / 16777216.0);
      a = __ddiv_rn(num, __dmul_rn(static_cast<double>(nq), m.norm));
      a = fmin(1.0, fmax(0.0, a));
    }
    // z = θ0 + θ_v v + θ_u u + θ_a a, left to right, no contraction (matches the oracle)
    double z = __dadd_rn(m.th0, __dmul_rn(m.thv, static_cast<double>(m.v[i])));
    z = __dadd_rn(z, __dmul_rn(m.thu, static_cast<double>(m.u[i])));
    z = __dadd_rn(z, __dmul_rn(m.tha, a));
    double sd = __ddiv_rn(1.0, __dadd_rn(1.0, exp(-z)));
    sd = fmin(1.0, fmax(0.0, sd));
    s = __double2float_rn(sd);
    af = static_cast<float>(a);
    m.s_state[i] = s;
  }
  m.a_out[i] = af;
  if (m.s_out) m.s_out[i] = m.open[i] ? 0.5f : s;
}

// ---------------------------------------------------------------- fused a2 + a3 (one launch)
// One CTA per (layer, KV head) row: (1) apply the fused score pass to every visible chunk of
// the row (as score_apply_kernel), (2) after a CTA barrier, the row's fp64 span sums of A
// for the listed closed nodes → Q = round-half-even(m·2^24), added to an int64 accumulator
// (integer addition: exact and order-independent, so the result equals the two-kernel path
// bit for bit); (3) the last CTA to finish (threadfence + ticket) publishes Mass and Mclose
// into mass2, resets the accumulators and — single rank — evaluates the MSVE score (a3).
struct FusedArgs {
  ApplyArgs ap;
  const int32_t *mass_nodes;
  int n_mass, N, L, H;
  SliceView sv;                // rows whose masses count (thin slice)
  int64_t max_tokens;
  const int32_t *nlen;
  unsigned long long *acc;     // [max_nodes] int64 accumulators (zero between calls)
  int64_t *mass_part, *mass2;
  const int64_t *mclose;
  unsigned int *ticket;
  unsigned int *row_done;      // [L·H] parts of each row past step (1) (zero at rest)
  long long *trace;            // ARBOR_POST_TRACE=1 (diagnostics): [CTA][16] globaltimer ns
  int do_msve;
  MsveArgs m;
};

#ifndef ARBOR_POST_THREADS
#define ARBOR_POST_THREADS 256
#endif
constexpr int kFusedThreads = ARBOR_POST_THREADS;

// the phase timeline (ARBOR_POST_TRACE=1 at run time) is compiled only into diagnostic builds
// (-DARBOR_POST_TRACE_BUILD)
#ifdef ARBOR_POST_TRACE_BUILD
constexpr bool kPostTrace = true;
#else
constexpr bool kPostTrace = false;
#endif
#define POST_TRACE(f, e)                                                                    \
  do {                                                                                      \
    if (kPostTrace && (f).trace && threadIdx.x == 0) {                                      \
      unsigned long long t_;                                                                \
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t_));                                \
      (f).trace[(static_cast<int64_t>(blockIdx.y) * gridDim.x + blockIdx.x) * 16 + (e)] =   \
          static_cast<long long>(t_);                                                       \
    }                                                                                       \
  } while (0)

// MSVE of node i from its inputs (open flag, Nq, Mass, Mclose, v, u): a_i, s_i (fp64, no
// contraction, same expression order as msve_kernel and the oracle)
__device__ __forceinline__ void msve_compute(const MsveArgs &m, int i, bool open, long long nq,
                                             long long mass, long long mclose, float v, float u) {
  float s = 0.5f, af = 0.f;
  if (!open) {
    double a = 0.0;
    if (nq > 0) {
      const double num = static_cast<double>(mass - mclose) * (1.0 / 16777216.0);
      a = __ddiv_rn(num, __dmul_rn(static_cast<double>(nq), m.norm));
      a = fmin(1.0, fmax(0.0, a));
    }
    double z = __dadd_rn(m.th0, __dmul_rn(m.thv, static_cast<double>(v)));
    z = __dadd_rn(z, __dmul_rn(m.thu, static_cast<double>(u)));
    z = __dadd_rn(z, __dmul_rn(m.tha, a));
    double sd = __ddiv_rn(1.0, __dadd_rn(1.0, exp(-z)));
    sd = fmin(1.0, fmax(0.0, sd));
    s = __double2float_rn(sd);
    af = static_cast<float>(a);
    m.s_state[i] = s;
  }
  m.a_out[i] = af;
  if (m.s_out) m.s_out[i] = open ? 0.5f : s;
}

// Steps (1)-(3) of one (row, part) CTA; lse2(b, g) gives the log2-domain LSE of leaf b's
// query head g of this row's KV head (the caller's LSE buffer, or the merged one in smem).
// Per-lane metadata of one batch of chunks (lane i: chunk w + NW·i of warp w) and of mass
// nodes (lane i: mass node w + NW·i).  Plan arrays, k_cur, n and spans are not written by
// the attention kernel, so decode_post loads the first batch before griddepcontrol.wait.
struct ChunkMeta {
  int node = 0, c0 = 0, p0 = 0, pc = 0, nt = 0, ident = 0;   // nt: chunk_span of the chunk
  long long sp = 0;
};
struct MassMeta {
  int node = 0, n = 0;
  long long sp = 0;
};
// chunk v of part `part`: plan chunk part + nparts·v (round robin: the shared root chunks
// spread over the parts)
__device__ __forceinline__ ChunkMeta load_chunk_meta(const FusedArgs &f, int v, int part,
                                                     int nparts) {
  const ApplyArgs &a = f.ap;
  ChunkMeta m;
  const int cm = part + nparts * v;
  if (cm < a.pv.C) {
    m.node = a.pv.ch_node[cm];
    m.c0 = a.pv.ch_chunk[cm] * kAttnChunk;
    m.p0 = a.pv.ch_poff[cm];
    m.pc = a.pv.ch_pcnt[cm];
    // A_i(t) = Σ_{u>b_i}: the open block that holds the query (an open active leaf)
    // gets no mass from it — its chunks attend but are skipped here (Q5')
    if (!f.m.open[m.node]) {
      const int kc = a.kcur[m.node], so = a.soff[m.node];
      m.nt = chunk_span(so, kc, m.c0, kAttnChunk);
      m.ident = kc == f.nlen[m.node] && so == 0;
      m.sp = a.span[m.node];
    }
  }
  return m;
}
__device__ __forceinline__ MassMeta load_mass_meta(const FusedArgs &f, int mm) {
  MassMeta m;
  if (mm < f.n_mass) {
    m.node = f.mass_nodes[mm];
    m.n = f.nlen[m.node];
    m.sp = f.ap.span[m.node];
  }
  return m;
}

template <typename LseFn>
__device__ __forceinline__ void score_row(const FusedArgs &f, int li, int h, int part, int nparts,
                                          LseFn lse2, const ChunkMeta *pre_c = nullptr,
                                          const MassMeta *pre_m = nullptr) {
  // (row, part): the part's chunks (round robin over the row's plan chunks) in step (1); the
  // row's last part to finish (1) computes every listed node's mass of the row in step (2)
  const ApplyArgs &a = f.ap;
  const int tid = threadIdx.x;
  // (1) A[li][h][a_j + pos] += Σ_pairs Σ_g exp2(z − LSE·log2 e)
  // A full node (k_cur = n) holds its tokens in position order (appends and rehydration
  // write the identity; only an eviction permutes slots, and it lowers k_cur), so its pos
  // tag is the slot itself: no page-table / tag round trip.  The pair loop's loads are
  // issued together (G ≤ 8 logits and LSEs per pair).
  const int warp = tid >> 5, lane = tid & 31;
  constexpr int NW = kFusedThreads / 32;
  const int lgP = 31 - __clz(a.g.P);
  // Warp w takes chunks w, w + NW, …  Their metadata is loaded 32 chunks at a time, lane i
  // holding chunk w + NW·i (two round trips per batch instead of two per chunk), then
  // broadcast chunk by chunk.
  const int Cp = a.pv.C > part ? (a.pv.C - part + nparts - 1) / nparts : 0;   // this part's chunks
  for (int cb = warp; cb < Cp; cb += NW * 32) {
    const ChunkMeta cmeta = (cb == warp && pre_c) ? *pre_c : load_chunk_meta(f, cb + NW * lane, part, nparts);
    const int m_node = cmeta.node, m_c0 = cmeta.c0, m_p0 = cmeta.p0, m_pc = cmeta.pc,
              m_nt = cmeta.nt, m_ident = cmeta.ident;
    const long long m_sp = cmeta.sp;
    const int nb = min(32, (Cp - cb + NW - 1) / NW);
    for (int j = 0; j < nb; ++j) {
      const int nt = __shfl_sync(0xffffffffu, m_nt, j);
      if (nt == 0) continue;
      const int node = __shfl_sync(0xffffffffu, m_node, j);
      const int c0 = __shfl_sync(0xffffffffu, m_c0, j);
      const int p0 = __shfl_sync(0xffffffffu, m_p0, j);
      const int pc = __shfl_sync(0xffffffffu, m_pc, j);
      const bool ident = __shfl_sync(0xffffffffu, m_ident, j) != 0;
      const int64_t sp = __shfl_sync(0xffffffffu, m_sp, j);
      const int32_t *pl = a.ptab + static_cast<int64_t>(node) * a.g.MPN;
      // both 32-slot halves of the chunk at once (lane: slots lane and lane + 32), so their
      // logit and A loads are in flight together
      const int hi = span_hi(nt), lo = span_lo(nt);   // valid slots [lo, hi) of the chunk (Q23*)
      const bool v0 = lane >= lo && lane < hi, v1 = lane + 32 >= lo && lane + 32 < hi;
      auto pos_of = [&](int slot) {   // page size: a power of two (arbor_init)
        return ident ? slot : a.pos[pool_row(a.g, li, pl[slot >> lgP], h, slot & (a.g.P - 1))];
      };
      float *Ar = a.A + (static_cast<int64_t>(li) * a.g.H + h) * a.g.max_tokens + sp;
      float *dst0 = v0 ? Ar + pos_of(c0 + lane) : nullptr;
      float *dst1 = v1 ? Ar + pos_of(c0 + lane + 32) : nullptr;
      const float old0 = v0 ? *dst0 : 0.f, old1 = v1 ? *dst1 : 0.f;
      // Σ over pairs (ascending) and query heads (ascending) per slot; four pairs' logits and
      // LSEs are loaded before any is used (the sum order is unchanged)
      float ps0 = 0.f, ps1 = 0.f;
      const int pe = p0 + pc;
      int p = p0;
      auto zrow = [&](int pp) {
        return a.zbuf + (((static_cast<int64_t>(pp) * a.Lc + li) * a.g.H + h) * a.G) * kAttnChunk + lane;
      };
      if (a.G <= 4) {
        for (; p + 4 <= pe; p += 4) {
          float z0[4][4], z1[4][4], ll[4][4];
#pragma unroll
          for (int u = 0; u < 4; ++u) {
            const int b = a.pv.pair_b[p + u];
            const float *z = zrow(p + u);
#pragma unroll
            for (int g = 0; g < 4; ++g) {
              if (g < a.G) {
                z0[u][g] = v0 ? z[g * kAttnChunk] : 0.f;
                z1[u][g] = v1 ? z[g * kAttnChunk + 32] : 0.f;
                ll[u][g] = lse2(b, g);
              }
            }
          }
#pragma unroll
          for (int u = 0; u < 4; ++u)
#pragma unroll
            for (int g = 0; g < 4; ++g)
              if (g < a.G) {
                ps0 += exp2f(z0[u][g] - ll[u][g]);
                ps1 += exp2f(z1[u][g] - ll[u][g]);
              }
        }
      }
      for (; p < pe; ++p) {
        const int b = a.pv.pair_b[p];
        const float *z = zrow(p);
        for (int g0 = 0; g0 < a.G; g0 += 8) {
          float z0[8], z1[8], ll[8];
#pragma unroll
          for (int g = 0; g < 8; ++g) {
            if (g0 + g < a.G) {
              z0[g] = v0 ? z[(g0 + g) * kAttnChunk] : 0.f;
              z1[g] = v1 ? z[(g0 + g) * kAttnChunk + 32] : 0.f;
              ll[g] = lse2(b, g0 + g);
            }
          }
#pragma unroll
          for (int g = 0; g < 8; ++g)
            if (g0 + g < a.G) {
              ps0 += exp2f(z0[g] - ll[g]);
              ps1 += exp2f(z1[g] - ll[g]);
            }
        }
      }
      if (v0) {
        const float nv = old0 + ps0;
        if (!(nv >= 0.f) || isinf(nv)) atomicOr(&a.ctrl->err, DERR_INVARIANT);
        *dst0 = nv;
      }
      if (v1) {
        const float nv = old1 + ps1;
        if (!(nv >= 0.f) || isinf(nv)) atomicOr(&a.ctrl->err, DERR_INVARIANT);
        *dst1 = nv;
      }
    }
  }
  POST_TRACE(f, 4);
  // row ticket: the last part of the row to get here sees every part's A updates
  __shared__ bool row_last;
  if (nparts > 1) {
    __threadfence();
    __syncthreads();
    if (tid == 0) {
      const int row = li * f.H + h;
      row_last = atomicAdd(&f.row_done[row], 1u) == static_cast<unsigned>(nparts - 1);
      if (row_last) f.row_done[row] = 0u;
    }
    __syncthreads();
    __threadfence();
  } else {
    __syncthreads();
    if (tid == 0) row_last = true;
    __syncthreads();
  }
  // (2) this row's partial node masses: warp per node, lanes strided, fixed xor tree (Q29);
  // node metadata batched like the chunks'.  Rows outside the thin slice add nothing.
  const float *Arow = a.A + (static_cast<int64_t>(li) * f.H + h) * f.max_tokens;
  POST_TRACE(f, 5);
  const int mass_end = (f.sv.has(li, h) && row_last) ? f.n_mass : 0;
  for (int mb = warp; mb < mass_end; mb += NW * 32) {
    const MassMeta mmeta = (mb == warp && pre_m) ? *pre_m : load_mass_meta(f, mb + NW * lane);
    const int m_node = mmeta.node, m_n = mmeta.n;
    const long long m_sp = mmeta.sp;
    const int nb = min(32, (mass_end - mb + NW - 1) / NW);
    for (int j = 0; j < nb; ++j) {
      const int n = __shfl_sync(0xffffffffu, m_n, j);
      if (n == 0) continue;
      const int node = __shfl_sync(0xffffffffu, m_node, j);
      const float *r = Arow + __shfl_sync(0xffffffffu, m_sp, j);
      double m = 0.0;
      for (int t = lane; t < n; t += 32) m += static_cast<double>(r[t]);
#pragma unroll
      for (int o = 16; o; o >>= 1) m += __shfl_xor_sync(0xffffffffu, m, o);
      if (lane == 0) atomicAdd(&f.acc[node], static_cast<unsigned long long>(__double2ll_rn(m * 16777216.0)));
    }
  }
  // (3) last CTA: publish, reset, MSVE.  Thread t owns nodes t, t + 256, …: the listed
  // (recomputed) ones take the accumulated sum, the rest keep their cached partial mass.
  // The inputs of each thread's first node and the listed-node bitmap are loaded before
  // the ticket (plan data and library state this kernel does not write), so the last CTA's
  // serial tail is one round trip (the accumulators) plus the MSVE arithmetic.
  POST_TRACE(f, 6);
  constexpr int kMaxNodes = 3072;                      // arbor_init's max_nodes bound
  __shared__ unsigned listed[kMaxNodes / 32];
  __shared__ bool last;
  for (int w = tid; w < (f.N + 31) / 32; w += kFusedThreads) listed[w] = 0u;
  const int i0 = tid;
  bool p_open = true;
  long long p_nq = 0, p_part = 0, p_mclose = 0;
  float p_v = 0.f, p_u = 0.f;
  if (i0 < f.N) {
    p_open = f.m.open[i0] != 0;
    p_nq = f.m.nq[i0];
    p_part = f.mass_part[i0];
    p_mclose = f.mclose[i0];
    p_v = f.m.v[i0];
    p_u = f.m.u[i0];
  }
  __syncthreads();
  for (int mi = tid; mi < f.n_mass; mi += kFusedThreads) {
    const int node = f.mass_nodes[mi];
    atomicOr(&listed[node >> 5], 1u << (node & 31));
  }
  __threadfence();
  __syncthreads();
  if (tid == 0) last = atomicAdd(f.ticket, 1u) == gridDim.x * gridDim.y - 1;
  __syncthreads();
  POST_TRACE(f, 7);
  if (!last) return;
  __threadfence();
  if (tid == 0) *f.ticket = 0u;
  for (int i = tid; i < f.N; i += kFusedThreads) {
    const bool first = i == i0;
    long long mass = first ? p_part : f.mass_part[i];
    if ((listed[i >> 5] >> (i & 31)) & 1u) {
      volatile unsigned long long *acc = f.acc;
      mass = static_cast<long long>(acc[i]);
      acc[i] = 0ull;
      f.mass_part[i] = mass;
    }
    const long long mclose = first ? p_mclose : f.mclose[i];
    f.mass2[i] = mass;
    f.mass2[f.N + i] = mclose;
    if (f.do_msve)
      msve_compute(f.m, i, first ? p_open : f.m.open[i] != 0, first ? p_nq : f.m.nq[i], mass,
                   mclose, first ? p_v : f.m.v[i], first ? p_u : f.m.u[i]);
  }
  __syncthreads();
  POST_TRACE(f, 8);
}

__global__ void __launch_bounds__(kFusedThreads)
score_fused_kernel(FusedArgs f) {
  pdl_wait();
  pdl_trigger();
  const int row = blockIdx.x;                        // li * H + h
  const int li = row / f.H, h = row - li * f.H;
  const float *ls = f.ap.lse + static_cast<int64_t>(li) * f.ap.Hq + h * f.ap.G;
  const int64_t bstride = static_cast<int64_t>(f.ap.Lc) * f.ap.Hq;
  // node-wise CTA ownership: node % gridDim.y
  score_row(f, li, h, blockIdx.y, gridDim.y,
            [&](int b, int g) { return ls[b * bstride + g] * kLog2e; });
}

// ---------------------------------------------------------------- f2: a9 merge + a2 + a3
// arbor_decode_step's second launch ("from attention weights already
// materialized during decoding"): one CTA per (row, part) first merges, root→leaf, the
// split-softmax partials the attention kernel left for every (active leaf b, query head g)
// of its row — M = max m, L = Σ 2^(m−M) l, o = Σ 2^(m−M) o_p / L, LSE₂ = M + log2 L (warp per
// (b, g), lanes over the path's pairs for M and L, over d for o) — keeps LSE₂ in shared
// memory, and then runs score_row on the logits with it.  Every part needs every LSE of the
// row, so M and L are computed by all parts (2 floats per pair), while o and the LSE output
// are written by part (b·G + g) mod parts only.  Replaces attn_merge_kernel + the score
// launch (and the LSE round trip through HBM) on the decode step.
struct PostArgs {
  FusedArgs f;
  const float *partials;
  void *out;
  float *lse_out;   // natural-log LSE, or NULL
  int nA;
  int exp;          // ARBOR_POST_EXP (measurement only): bit0 skip (b), bit1 skip score_row
};
constexpr int kPostItems = 512;   // nA · G ≤ kPostItems (host-checked)

template <typename T, int D, int MINB>
__global__ void __launch_bounds__(kFusedThreads, MINB)
decode_post_kernel(PostArgs pa) {
  const FusedArgs &f = pa.f;
  const ApplyArgs &a = f.ap;
  POST_TRACE(f, 0);
  const int row = blockIdx.x, part = blockIdx.y, nparts = gridDim.y;
  const int li = row / f.H, h = row - li * f.H;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  constexpr int NW = kFusedThreads / 32, EPL = D / 32;
// Prefetching score_row's first chunk / mass metadata here, before griddepcontrol.wait, kept
// ~11 registers live through phases (a) and (b) and spilled at the 128-register cap: without it
// C3 DPTS decode_post 66.9 -> 63.6 us, C2 17.4 -> 16.7 us (round 2, late; -DARBOR_POST_PREFETCH=1
// restores it)
#ifndef ARBOR_POST_PREFETCH
#define ARBOR_POST_PREFETCH 0
#endif
#if ARBOR_POST_PREFETCH
  const ChunkMeta pre_c = load_chunk_meta(f, warp + NW * lane, part, nparts);
  const MassMeta pre_m = load_mass_meta(f, warp + NW * lane);
#endif
  // … and the first (leaf, q head) item's path bounds and this lane's first pair (plan arrays)
  int pre_p0 = 0, pre_p1 = 0, pre_pi = 0;
  {
    const int it = threadIdx.x >> 3;
    if (it < pa.nA * a.G) {
      const int b = it / a.G;
      pre_p0 = a.pv.bp_off[b];
      pre_p1 = a.pv.bp_off[b + 1];
      if (pre_p0 + (lane & 7) < pre_p1) pre_pi = a.pv.bp_list[pre_p0 + (lane & 7)];
    }
  }
  pdl_wait();
  pdl_trigger();
  POST_TRACE(f, 1);
  const int G = a.G;
  __shared__ float lse2s[kPostItems], Ms[kPostItems], invL[kPostItems];
  auto part_ptr = [&](int p, int g) -> const float * {
    return pa.partials + (((static_cast<int64_t>(p) * a.Lc + li) * f.H + h) * G + g) * (D + 2);
  };
  const int nitems = pa.nA * G;
  // (a) eight lanes per (b, g): each lane folds every 8th pair of the leaf's path online
  // (M, L), the group combines them: M = max m, L = Σ 2^(m−M) l → LSE₂ = M + log2 L
  {
    const int sub = lane & 7;
    for (int it0 = (threadIdx.x >> 3); it0 < ((nitems + 3) & ~3); it0 += kFusedThreads / 8) {
      const int it = it0;
      const bool ok = it < nitems;
      const bool first = it0 == (threadIdx.x >> 3);   // prefetched before griddepcontrol.wait
      const int b = ok ? it / G : 0, g = ok ? it - b * G : 0;
      const int p0 = ok ? (first ? pre_p0 : a.pv.bp_off[b]) : 0;
      const int p1 = ok ? (first ? pre_p1 : a.pv.bp_off[b + 1]) : 0;
      float M = -INFINITY, Ls = 0.f;
      for (int i = p0 + sub; i < p1; i += 8) {
        const float *pp = part_ptr((first && i == p0 + sub) ? pre_pi : a.pv.bp_list[i], g);
        const float m2 = pp[D], l2 = pp[D + 1];
        if (m2 == -INFINITY) continue;
        if (m2 > M) {
          Ls = Ls * exp2f(M - m2) + l2;   // exp2(−inf) = 0 on the first pair
          M = m2;
        } else {
          Ls = fmaf(exp2f(m2 - M), l2, Ls);
        }
      }
#pragma unroll
      for (int o = 4; o; o >>= 1) {
        const float Mo = __shfl_xor_sync(0xffffffffu, M, o);
        const float Lo = __shfl_xor_sync(0xffffffffu, Ls, o);
        const float Mn = fmaxf(M, Mo);
        Ls = (Mn == -INFINITY) ? 0.f
             : (M == -INFINITY ? 0.f : Ls * exp2f(M - Mn)) + (Mo == -INFINITY ? 0.f : Lo * exp2f(Mo - Mn));
        M = Mn;
      }
      if (ok && sub == 0) {
        lse2s[it] = Ls > 0.f ? M + log2f(Ls) : -INFINITY;
        Ms[it] = M;
        invL[it] = Ls > 0.f ? 1.f / Ls : 0.f;
        if ((it & (nparts - 1)) == part && pa.lse_out)
          pa.lse_out[(static_cast<int64_t>(b) * a.Lc + li) * a.Hq + h * G + g] =
              Ls > 0.f ? (M + log2f(Ls)) * 0.6931471805599453f : -INFINITY;
      }
    }
  }
  __syncthreads();
  POST_TRACE(f, 2);
  // (b) owned items, eight lanes per item (four items per warp at once): lane j of the group
  // holds pair p0 + j's index and weight 2^(m−M); then, pairs in path order, each lane
  // accumulates D/8 of o with float2 loads: o = Σ w o_p / L
  {
    constexpr int EPG = D / 8;             // floats of o per lane
    const int sub = lane & 7, gbase = lane & ~7;
    const int nown = nitems > part ? (nitems - part + nparts - 1) / nparts : 0;   // owned items
    for (int o0 = warp * 4; o0 < ((pa.exp & 1) ? 0 : ((nown + 3) & ~3)); o0 += NW * 4) {
      const int oi = o0 + (lane >> 3);
      const bool ok = oi < nown;
      const int it = part + oi * nparts;
      const int b = ok ? it / G : 0, g = ok ? it - b * G : 0;
      const int p0 = ok ? a.pv.bp_off[b] : 0, p1 = ok ? a.pv.bp_off[b + 1] : 0;
      const float M = ok ? Ms[it] : -INFINITY;
      float acc[EPG];
#pragma unroll
      for (int e = 0; e < EPG; ++e) acc[e] = 0.f;
      const int np = p1 - p0;
      int npmax = max(np, __shfl_xor_sync(0xffffffffu, np, 8));     // max over the 4 groups
      npmax = max(npmax, __shfl_xor_sync(0xffffffffu, npmax, 16));
      for (int i0 = 0; i0 < npmax; i0 += 8) {
        int pi = 0;
        float w = 0.f;
        if (i0 + sub < np && M != -INFINITY) {
          pi = a.pv.bp_list[p0 + i0 + sub];
          const float m2 = part_ptr(pi, g)[D];
          w = m2 == -INFINITY ? 0.f : exp2f(m2 - M);
        }
#pragma unroll 2
        for (int j = 0; j < 8; ++j) {
          const float wj = __shfl_sync(0xffffffffu, w, gbase + j);
          const int pj = __shfl_sync(0xffffffffu, pi, gbase + j);
          const float2 *pp = reinterpret_cast<const float2 *>(part_ptr(pj, g)) + sub * (EPG / 2);
          float2 v[EPG / 2];
#pragma unroll
          for (int e = 0; e < EPG / 2; ++e) v[e] = pp[e];
          if (wj != 0.f) {
#pragma unroll
            for (int e = 0; e < EPG / 2; ++e) {
              acc[2 * e] = fmaf(wj, v[e].x, acc[2 * e]);
              acc[2 * e + 1] = fmaf(wj, v[e].y, acc[2 * e + 1]);
            }
          }
        }
      }
      if (ok) {
        T *out = static_cast<T *>(pa.out) + ((static_cast<int64_t>(b) * a.Lc + li) * a.Hq + h * G + g) * D +
                 sub * EPG;
        const float inv = invL[it];
#pragma unroll
        for (int e = 0; e < EPG; ++e) out[e] = ElemT<T>::from_f(acc[e] * inv);
      }
    }
  }
  __syncthreads();
  POST_TRACE(f, 3);
  if (pa.exp & 2) return;
#if ARBOR_POST_PREFETCH
  score_row(f, li, h, part, nparts, [&](int b, int g) { return lse2s[b * G + g]; }, &pre_c, &pre_m);
#else
  score_row(f, li, h, part, nparts, [&](int b, int g) { return lse2s[b * G + g]; });
#endif
}

}  // namespace

long long *g_post_trace = nullptr;
size_t g_post_trace_n = 0;

namespace {
FusedArgs fused_args(arbor_ctx *c, const PlanView &pv, const float *lse, const int32_t *d_nodes,
                     int num_nodes, int N, bool do_msve, float *s_out) {
  FusedArgs f{};
  ApplyArgs &a = f.ap;
  a.pv = pv;
  a.g = PoolView{c->L, c->H, c->P, c->D, c->NP, c->max_pages_node, c->max_tokens};
  a.pos = c->cfg.pos_pool;
  a.ptab = c->d.ptab;
  a.kcur = c->d.kcur;
  a.soff = c->d.soff;
  a.span = c->d.span;
  a.zbuf = c->d.zbuf;
  a.lse = lse;
  a.A = c->cfg.score;
  a.ctrl = c->d.ctrl;
  a.Lc = c->L;
  a.Hq = c->Hq;
  a.G = c->G;
  f.sv = slice_view(c);
  f.mass_nodes = d_nodes;
  f.n_mass = num_nodes;
  f.N = N;
  f.L = c->L;
  f.H = c->H;
  f.max_tokens = c->max_tokens;
  f.nlen = c->d.n;
  f.acc = reinterpret_cast<unsigned long long *>(c->d.mass_acc);
  f.mass_part = c->d.mass_part;
  f.mass2 = c->d.mass2;
  f.mclose = c->d.mclose;
  f.ticket = c->d.ticket;
  f.row_done = c->d.row_done;
  f.trace = nullptr;
  if (getenv("ARBOR_POST_TRACE")) {
    const size_t need = static_cast<size_t>(c->L) * c->H * 64 * 16;
    if (need > g_post_trace_n) {
      if (g_post_trace) cudaFree(g_post_trace);
      cudaMalloc(&g_post_trace, need * sizeof(long long));
      g_post_trace_n = need;
    }
    cudaMemsetAsync(g_post_trace, 0, g_post_trace_n * sizeof(long long), c->ms);
    f.trace = g_post_trace;
  }
  f.do_msve = do_msve ? 1 : 0;
  MsveArgs &m = f.m;
  m.N = N;
  m.open = c->d.open;
  m.v = c->d.v;
  m.u = c->d.u;
  m.mass2 = c->d.mass2;
  m.nq = c->nq_dev ? c->nq_dev : c->d.nq;
  m.norm = msve_norm(c);
  m.th0 = c->prm.theta[0];
  m.thv = c->prm.theta[1];
  m.thu = c->prm.theta[2];
  m.tha = c->prm.theta[3];
  m.a_out = c->d.a;
  m.s_state = c->d.s;
  m.s_out = s_out;
  return f;
}
}  // namespace

void launch_score_fused(arbor_ctx *c, const PlanView &pv, const float *lse, const int32_t *d_nodes,
                        int num_nodes, int N, bool do_msve, float *s_out, int nparts) {
  const FusedArgs f = fused_args(c, pv, lse, d_nodes, num_nodes, N, do_msve, s_out);
  stage_begin(c, ARBOR_ST_SCORE_ACCUM, c->ms);
  launch_pdl(score_fused_kernel, dim3(c->L * c->H, nparts), dim3(kFusedThreads), 0, c->ms, f);
  ARBOR_LAUNCHED(c);
  stage_end(c, ARBOR_ST_SCORE_ACCUM, c->ms);
}

bool decode_post_fits(arbor_ctx *c, int nA) { return nA * c->G <= kPostItems; }

void launch_decode_post(arbor_ctx *c, const PlanView &pv, void *out, float *lse_out,
                        const int32_t *d_nodes, int num_nodes, int N, bool do_msve, float *s_out,
                        int nparts) {
  PostArgs pa{};
  pa.f = fused_args(c, pv, nullptr, d_nodes, num_nodes, N, do_msve, s_out);
  pa.partials = c->d.partials;
  pa.out = out;
  pa.lse_out = lse_out;
  pa.nA = pv.nA;
  static const int pexp = getenv("ARBOR_POST_EXP") ? atoi(getenv("ARBOR_POST_EXP")) : 0;
  pa.exp = pexp;
  const dim3 grid(c->L * c->H, nparts);
  stage_begin(c, ARBOR_ST_SCORE_ACCUM, c->ms);
  // PDL launch.  (An earlier version — 2 CTAs per row, 110 registers, no min-blocks bound —
  // was slower as a PDL launch than as a plain one, 269 vs 237 µs per C2 step; this one is
  // faster with PDL: 238.9 vs 243.7 µs, A/B on one box.)
  if (c->esize == 2) {
    if (c->D == 128) launch_pdl(decode_post_kernel<__nv_bfloat16, 128, kPostCtasPerSm>, grid, dim3(kFusedThreads), 0, c->ms, pa);
    else launch_pdl(decode_post_kernel<__nv_bfloat16, 64, kPostCtasPerSm>, grid, dim3(kFusedThreads), 0, c->ms, pa);
  } else {
    if (c->D == 128) launch_pdl(decode_post_kernel<float, 128, kPostCtasPerSm>, grid, dim3(kFusedThreads), 0, c->ms, pa);
    else launch_pdl(decode_post_kernel<float, 64, kPostCtasPerSm>, grid, dim3(kFusedThreads), 0, c->ms, pa);
  }
  ARBOR_LAUNCHED(c);
  stage_end(c, ARBOR_ST_SCORE_ACCUM, c->ms);
}

void launch_node_mass(arbor_ctx *c, const int32_t *d_nodes, int num_nodes, int64_t *out,
                      int out_stride) {
  if (num_nodes == 0) return;
  node_mass_kernel<<<dim3(num_nodes, c->L), kMassThreads, 0, c->ms>>>(
      d_nodes, c->d.n, c->d.span, c->cfg.score, c->L, c->H, c->max_tokens, c->d.mass_scratch,
      slice_view(c));
  node_mass_finalize<<<(num_nodes + 127) / 128, 128, 0, c->ms>>>(d_nodes, num_nodes, c->L,
                                                                 c->d.mass_scratch, out, out_stride);
  c->launches += 2;
}

void launch_msve(arbor_ctx *c, int N, float *s_out) {
  MsveArgs m{};
  m.N = N;
  m.open = c->d.open;
  m.v = c->d.v;
  m.u = c->d.u;
  m.mass2 = c->d.mass2;
  m.nq = c->nq_dev ? c->nq_dev : c->d.nq;
  m.norm = msve_norm(c);
  m.th0 = c->prm.theta[0];
  m.thv = c->prm.theta[1];
  m.thu = c->prm.theta[2];
  m.tha = c->prm.theta[3];
  m.a_out = c->d.a;
  m.s_state = c->d.s;
  m.s_out = s_out;
  stage_begin(c, ARBOR_ST_MSVE, c->ms);
  msve_kernel<<<(N + 255) / 256, 256, 0, c->ms>>>(m);
  ARBOR_LAUNCHED(c);
  stage_end(c, ARBOR_ST_MSVE, c->ms);
}

}  // namespace arbor

// debug only (not part of include/arbor.h): the last ARBOR_POST_TRACE timeline of
// decode_post / score_fused ([CTA = part·rows + row][16] globaltimer ns: 0 start, 1 past
// griddepcontrol.wait, 2 (a) merged LSE, 3 (b) outputs, 4 (1) A updates, 5 row ticket,
// 6 (2) masses, 7 global ticket, 8 the last CTA's MSVE done)
extern "C" int arbor_debug_post_trace(long long *host, long long count) {
  if (!arbor::g_post_trace || count < 0 || static_cast<size_t>(count) > arbor::g_post_trace_n) return -1;
  cudaDeviceSynchronize();
  return cudaMemcpy(host, arbor::g_post_trace, sizeof(long long) * count, cudaMemcpyDeviceToHost) == cudaSuccess ? 0 : -2;
}
