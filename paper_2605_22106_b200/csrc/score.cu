// score.cu — §8(a) a2 (accumulated attention), a3 (node mass + MSVE).
//
// a2 (§4 Execution (iii)): A_i(t) = Σ_{u>b_i} Σ_l Σ_h Attn_{u→t}.  Per
// decode step and active leaf b: p_t = exp(q·k_t/√d − LSE_{b,l,g}) over the visible slots
// of Path(ℓ_b), A[l][h][a_j + pos_t] += Σ_{g∈group(h)} p_t.  One CTA owns a (segment,
// layer, KV head): it stages the segment's K rows once and sums the contributions of every
// active leaf sharing the node in ascending leaf order, then does a single read-modify-write
// of A per token — deterministic, no float atomics (Q30).
//
// a3 (Q4/Q5/Q29): m_{l,h,i} = Σ_{t∈span_i} A[l][h][t] accumulated in fp64,
// Q = round-half-even(m · 2^24) as int64, Mass_i = Σ_rows Q (exact int64 sums: order- and
// world-size-independent); a_i = clamp((Mass_i − Mclose_i) 2^-24 / (Nq_i L Hq), 0, 1);
// s_i = clip(σ(θ0 + θ_v v_i + θ_u u_i + θ_a a_i), 0, 1) in fp64, rounded to f32.
#include "tile.cuh"

namespace arbor {
namespace {

constexpr float kLog2e = 1.4426950408889634f;

struct ScoreArgs {
  PlanView pv;
  PoolView g;
  const void *kpool;
  const int16_t *pos;
  const int32_t *ptab, *kcur;
  const int64_t *span;
  const void *q;
  const float *lse;
  float *A;
  Ctrl *ctrl;
  int Lc, Hq, G, lb_per;
  float scale_log2;
};

template <typename T, int D, int QB>
__global__ void __launch_bounds__(128)
score_accum_kernel(ScoreArgs a) {
  constexpr int CH = kAttnChunk;
  const int s = blockIdx.x, li = blockIdx.y, h = blockIdx.z;
  const int node = a.pv.seg_node[s];
  const int c0 = a.pv.seg_chunk[s] * CH;
  const int nt = max(0, min(CH, a.kcur[node] - c0));
  if (nt == 0) return;
  const int loff = a.pv.seg_loff[s], lcnt = a.pv.seg_lcnt[s];
  const int G = a.G;
  extern __shared__ __align__(16) unsigned char sm[];
  T *Ks = reinterpret_cast<T *>(sm);
  int64_t *rowoff = reinterpret_cast<int64_t *>(Ks + CH * D);
  float *qs = reinterpret_cast<float *>(rowoff + CH);   // [QB][D]
  float *ls = qs + QB * D;                               // [QB] LSE·log2e
  const T *kpool = static_cast<const T *>(a.kpool);
  const T *q = static_cast<const T *>(a.q);
  stage_tile<T, D, false>(Ks, nullptr, rowoff, kpool, nullptr, a.ptab + node * a.g.MPN, c0, nt,
                          a.g, li, h);
  const int t = threadIdx.x;
  float psum = 0.f;
  for (int b0 = 0; b0 < lcnt; b0 += a.lb_per) {
    const int nb = min(a.lb_per, lcnt - b0);
    const int nq = nb * G;
    for (int idx = threadIdx.x; idx < nq * D; idx += blockDim.x) {
      const int qi = idx / D, e = idx - qi * D;
      const int bi = qi / G, g = qi - bi * G;
      const int b = a.pv.pair_b[loff + b0 + bi];
      qs[idx] = ElemT<T>::to_f(q[((static_cast<int64_t>(b) * a.Lc + li) * a.Hq + h * G + g) * D + e]);
    }
    for (int qi = threadIdx.x; qi < nq; qi += blockDim.x) {
      const int bi = qi / G, g = qi - bi * G;
      const int b = a.pv.pair_b[loff + b0 + bi];
      ls[qi] = a.lse[(static_cast<int64_t>(b) * a.Lc + li) * a.Hq + h * G + g] * kLog2e;
    }
    cp_async_wait_all();
    __syncthreads();
    if (t < nt) {
      float acc[QB];
      row_dots<T, D, QB>(Ks, qs, t, nq, acc);
#pragma unroll
      for (int qi = 0; qi < QB; ++qi)
        if (qi < nq) psum += exp2f(fmaf(acc[qi], a.scale_log2, -ls[qi]));
    }
    __syncthreads();
  }
  if (t < nt) {
    const int pos = a.pos[rowoff[t]];
    float *dst = a.A + (static_cast<int64_t>(li) * a.g.H + h) * a.g.max_tokens + a.span[node] + pos;
    const float nv = *dst + psum;
    if (!(nv >= 0.f) || isinf(nv)) atomicOr(&a.ctrl->err, DERR_INVARIANT);
    *dst = nv;
  }
}

template <typename T, int D, int QB>
void launch_score_t(arbor_ctx *c, const ScoreArgs &a, int S) {
  constexpr int CH = kAttnChunk;
  const size_t smem = CH * D * sizeof(T) + CH * sizeof(int64_t) + (QB * D + QB) * sizeof(float);
  static bool attr_set = false;
  if (!attr_set) {
    cudaFuncSetAttribute(score_accum_kernel<T, D, QB>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         static_cast<int>(smem));
    attr_set = true;
  }
  dim3 grid(S, c->L, c->H);
  score_accum_kernel<T, D, QB><<<grid, 128, smem, c->ms>>>(a);
}

template <typename T, int D>
void launch_score_q(arbor_ctx *c, ScoreArgs a, int S, int max_q) {
  int qb;
  if (max_q <= 4 && c->G <= 4) qb = 4;
  else if (max_q <= 8 && c->G <= 8) qb = 8;
  else if (max_q <= 16 && c->G <= 16) qb = 16;
  else qb = 32;
  a.lb_per = qb / a.G > 0 ? qb / a.G : 1;
  switch (qb) {
    case 4: launch_score_t<T, D, 4>(c, a, S); break;
    case 8: launch_score_t<T, D, 8>(c, a, S); break;
    case 16: launch_score_t<T, D, 16>(c, a, S); break;
    default: launch_score_t<T, D, 32>(c, a, S); break;
  }
}

// One CTA per listed node: warps stride over the local layers, each warp sums one
// (layer, head) row of A over the node's span in fp64 (lanes strided, xor-tree: fixed
// order), quantises Q = round-half-even(m · 2^24) and accumulates the int64 Q of its rows;
// the CTA reduces its warps' integers and writes Σ_rows Q to out[node * out_stride].
constexpr int kMassThreads = 256;
__global__ void __launch_bounds__(kMassThreads)
node_mass_kernel(const int32_t *__restrict__ nodes, const int32_t *__restrict__ nlen,
                 const int64_t *__restrict__ span, const float *__restrict__ A, int L, int H,
                 int64_t max_tokens, int64_t *__restrict__ out, int out_stride) {
  const int node = nodes[blockIdx.x];
  const int n = nlen[node];
  const int64_t a0 = span[node];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  constexpr int kW = kMassThreads / 32;
  __shared__ long long red[kW];
  long long qsum = 0;
  for (int r = warp; r < L * H; r += kW) {
    const float *row = A + static_cast<int64_t>(r) * max_tokens + a0;
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
    out[static_cast<int64_t>(node) * out_stride] = tot;
  }
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

}  // namespace

void launch_score_accum(arbor_ctx *c, const PlanView &pv, int max_q, const void *q,
                        const float *lse, int layer_count) {
  if (pv.S == 0) return;
  ScoreArgs a{};
  a.pv = pv;
  a.g = PoolView{c->L, c->H, c->P, c->D, c->NP, c->max_pages_node, c->max_tokens};
  a.kpool = c->cfg.k_pool;
  a.pos = c->cfg.pos_pool;
  a.ptab = c->d.ptab;
  a.kcur = c->d.kcur;
  a.span = c->d.span;
  a.q = q;
  a.lse = lse;
  a.A = c->cfg.score;
  a.ctrl = c->d.ctrl;
  a.Lc = layer_count;
  a.Hq = c->Hq;
  a.G = c->G;
  a.scale_log2 = kLog2e / sqrtf(static_cast<float>(c->D));
  stage_begin(c, ARBOR_ST_SCORE_ACCUM, c->ms);
  if (c->esize == 2) {
    if (c->D == 128) launch_score_q<__nv_bfloat16, 128>(c, a, pv.S, max_q);
    else launch_score_q<__nv_bfloat16, 64>(c, a, pv.S, max_q);
  } else {
    if (c->D == 128) launch_score_q<float, 128>(c, a, pv.S, max_q);
    else launch_score_q<float, 64>(c, a, pv.S, max_q);
  }
  ARBOR_LAUNCHED(c);
  stage_end(c, ARBOR_ST_SCORE_ACCUM, c->ms);
}

void launch_node_mass(arbor_ctx *c, const int32_t *d_nodes, int num_nodes, int64_t *out,
                      int out_stride) {
  if (num_nodes == 0) return;
  node_mass_kernel<<<num_nodes, kMassThreads, 0, c->ms>>>(d_nodes, c->d.n, c->d.span,
                                                          c->cfg.score, c->L, c->H,
                                                          c->max_tokens, out, out_stride);
  ARBOR_LAUNCHED(c);
}

void launch_msve(arbor_ctx *c, int N, float *s_out) {
  MsveArgs m{};
  m.N = N;
  m.open = c->d.open;
  m.v = c->d.v;
  m.u = c->d.u;
  m.mass2 = c->d.mass2;
  m.nq = c->d.nq;
  m.norm = static_cast<double>(c->Lg) * static_cast<double>(c->Hqg);
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
