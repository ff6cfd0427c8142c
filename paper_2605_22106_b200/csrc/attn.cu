// attn.cu — §8(a) a9: tree decode attention over the compacted ancestor-path pages.
//
// PAPER.md P:63 ("next-token decoding depends exclusively on the ancestor chain of the
// active leaf").  For every active leaf b, layer l and query head g
// (KV head h = g / G, Q24):  o = Σ_t softmax_t(q·k_t/√d) v_t over the retained slots of
// Path(ℓ_b), root→leaf; LSE = ln Σ_t exp(q·k_t/√d).
//
// B200 design: one CTA per (segment = node × 128-slot chunk of the union of the active
// paths, layer, KV head).  The segment's K and V rows are staged once into shared memory
// with cp.async (16-byte, coalesced, K XOR-swizzled) and reused by EVERY active leaf whose
// path contains the node and by all G query heads of the KV head (tree sharing: a node
// shared by n leaves is read from HBM once).  Each CTA emits split-softmax partials
// (o·e^{-m}, m, Σe^{z-m}) in the log2 domain; a merge kernel combines a leaf's partials in
// a fixed root→leaf order (deterministic, no float atomics).
#include <cfloat>

#include "tile.cuh"

namespace arbor {
namespace {

constexpr float kLog2e = 1.4426950408889634f;
constexpr float kLn2 = 0.6931471805599453f;

struct AttnArgs {
  PlanView pv;
  PoolView g;
  const void *kpool, *vpool;
  const int32_t *ptab, *kcur;
  const void *q;
  float *partials;
  int layer_begin, Lc, Hq, G, lb_per;
  float scale_log2;   // log2(e)/sqrt(d)
};

template <typename T, int D, int QB>
__global__ void __launch_bounds__(128)
attn_partial_kernel(AttnArgs a) {
  constexpr int CH = kAttnChunk;
  constexpr int NCP = D / 2;        // column pairs in the PV phase
  constexpr int TG = 128 / NCP;     // token groups in the PV phase
  const int s = blockIdx.x, li = blockIdx.y, h = blockIdx.z;
  const int l = a.layer_begin + li;
  const int node = a.pv.seg_node[s];
  const int c0 = a.pv.seg_chunk[s] * CH;
  const int nt = max(0, min(CH, a.kcur[node] - c0));
  const int loff = a.pv.seg_loff[s], lcnt = a.pv.seg_lcnt[s];
  const int G = a.G;

  extern __shared__ __align__(16) unsigned char sm[];
  T *Ks = reinterpret_cast<T *>(sm);
  T *Vs = Ks + CH * D;
  int64_t *rowoff = reinterpret_cast<int64_t *>(Vs + CH * D);
  float *qs = reinterpret_cast<float *>(rowoff + CH);   // [QB][D]
  float *zs = qs + QB * D;                               // [QB][CH]
  float *os = zs + QB * CH;                              // [TG][QB][D]
  float *mls = os + TG * QB * D;                         // m2[QB], l[QB]

  const T *kpool = static_cast<const T *>(a.kpool);
  const T *vpool = static_cast<const T *>(a.vpool);
  const T *q = static_cast<const T *>(a.q);
  if (nt > 0)
    stage_tile<T, D, true>(Ks, Vs, rowoff, kpool, vpool, a.ptab + node * a.g.MPN, c0, nt, a.g,
                           l, h);

  for (int b0 = 0; b0 < lcnt; b0 += a.lb_per) {
    const int nb = min(a.lb_per, lcnt - b0);
    const int nq = nb * G;
    for (int idx = threadIdx.x; idx < nq * D; idx += blockDim.x) {
      const int qi = idx / D, e = idx - qi * D;
      const int bi = qi / G, g = qi - bi * G;
      const int b = a.pv.pair_b[loff + b0 + bi];
      qs[idx] = ElemT<T>::to_f(q[((static_cast<int64_t>(b) * a.Lc + li) * a.Hq + h * G + g) * D + e]);
    }
    cp_async_wait_all();
    __syncthreads();
    if (nt == 0) {
      for (int idx = threadIdx.x; idx < nq * (D + 2); idx += blockDim.x) {
        const int qi = idx / (D + 2), e = idx - qi * (D + 2);
        const int bi = qi / G, g = qi - bi * G;
        float *dst = a.partials +
                     ((((static_cast<int64_t>(loff + b0 + bi)) * a.Lc + li) * a.g.H + h) * G + g) *
                         (D + 2);
        dst[e] = (e == D) ? -INFINITY : 0.f;
      }
      __syncthreads();
      continue;
    }
    // phase 1: z = q·k (log2 domain), thread per token
    {
      const int t = threadIdx.x;
      if (t < nt) {
        float acc[QB];
        row_dots<T, D, QB>(Ks, qs, t, nq, acc);
#pragma unroll
        for (int qi = 0; qi < QB; ++qi)
          if (qi < nq) zs[qi * CH + t] = acc[qi] * a.scale_log2;
      } else {
        for (int qi = 0; qi < nq; ++qi) zs[qi * CH + t] = -INFINITY;
      }
    }
    __syncthreads();
    // phase 2: per-query max and exp-sum over the chunk (warp per query row)
    {
      const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
      for (int qi = w; qi < nq; qi += 4) {
        float v[CH / 32];
        float m = -INFINITY;
#pragma unroll
        for (int j = 0; j < CH / 32; ++j) {
          v[j] = zs[qi * CH + lane + 32 * j];
          m = fmaxf(m, v[j]);
        }
#pragma unroll
        for (int o = 16; o; o >>= 1) m = fmaxf(m, __shfl_xor_sync(0xffffffffu, m, o));
        float sum = 0.f;
#pragma unroll
        for (int j = 0; j < CH / 32; ++j) {
          const float p = (v[j] == -INFINITY) ? 0.f : exp2f(v[j] - m);
          zs[qi * CH + lane + 32 * j] = p;
          sum += p;
        }
#pragma unroll
        for (int o = 16; o; o >>= 1) sum += __shfl_xor_sync(0xffffffffu, sum, o);
        if (lane == 0) {
          mls[qi] = m;
          mls[QB + qi] = sum;
        }
      }
    }
    __syncthreads();
    // phase 3: o = Σ_t p_t v_t; thread = (column pair, token group)
    {
      const int cp = threadIdx.x % NCP, tg = threadIdx.x / NCP;
      float acc[QB][2];
#pragma unroll
      for (int qi = 0; qi < QB; ++qi) acc[qi][0] = acc[qi][1] = 0.f;
      for (int t = tg; t < nt; t += TG) {
        const float2 vf = ElemT<T>::ld2(Vs + t * D + 2 * cp);
#pragma unroll
        for (int qi = 0; qi < QB; ++qi) {
          if (qi < nq) {
            const float p = zs[qi * CH + t];
            acc[qi][0] = fmaf(p, vf.x, acc[qi][0]);
            acc[qi][1] = fmaf(p, vf.y, acc[qi][1]);
          }
        }
      }
#pragma unroll
      for (int qi = 0; qi < QB; ++qi) {
        if (qi < nq) {
          os[(tg * QB + qi) * D + 2 * cp] = acc[qi][0];
          os[(tg * QB + qi) * D + 2 * cp + 1] = acc[qi][1];
        }
      }
    }
    __syncthreads();
    for (int idx = threadIdx.x; idx < nq * (D + 2); idx += blockDim.x) {
      const int qi = idx / (D + 2), e = idx - qi * (D + 2);
      const int bi = qi / G, g = qi - bi * G;
      float val;
      if (e < D) {
        val = 0.f;
#pragma unroll
        for (int j = 0; j < TG; ++j) val += os[(j * QB + qi) * D + e];
      } else {
        val = mls[(e - D) * QB + qi];
      }
      a.partials[((((static_cast<int64_t>(loff + b0 + bi)) * a.Lc + li) * a.g.H + h) * G + g) *
                     (D + 2) + e] = val;
    }
    __syncthreads();
  }
}

struct MergeArgs {
  PlanView pv;
  const float *partials;
  void *out;
  float *lse;
  int Lc, Hq, G, H;
};

// One warp per (leaf b, layer, q head): combine the leaf's path partials root→leaf.
template <typename T, int D>
__global__ void __launch_bounds__(128)
attn_merge_kernel(MergeArgs a) {
  const int wid = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  const int total = a.pv.nA * a.Lc * a.Hq;
  if (wid >= total) return;
  const int gq = wid % a.Hq;
  const int li = (wid / a.Hq) % a.Lc;
  const int b = wid / (a.Hq * a.Lc);
  const int h = gq / a.G, g = gq - h * a.G;
  const int p0 = a.pv.bp_off[b], p1 = a.pv.bp_off[b + 1];
  constexpr int EPL = D / 32;
  auto part = [&](int p) -> const float * {
    return a.partials + ((((static_cast<int64_t>(p)) * a.Lc + li) * a.H + h) * a.G + g) * (D + 2);
  };
  float M = -INFINITY;
  for (int i = p0; i < p1; ++i) M = fmaxf(M, part(a.pv.bp_list[i])[D]);
  float acc[EPL];
#pragma unroll
  for (int j = 0; j < EPL; ++j) acc[j] = 0.f;
  float Ls = 0.f;
  if (M != -INFINITY) {
    for (int i = p0; i < p1; ++i) {
      const float *pp = part(a.pv.bp_list[i]);
      const float m2 = pp[D];
      if (m2 == -INFINITY) continue;
      const float w = exp2f(m2 - M);
      Ls = fmaf(w, pp[D + 1], Ls);
#pragma unroll
      for (int j = 0; j < EPL; ++j) acc[j] = fmaf(w, pp[lane + 32 * j], acc[j]);
    }
  }
  T *out = static_cast<T *>(a.out) + ((static_cast<int64_t>(b) * a.Lc + li) * a.Hq + gq) * D;
  const float inv = (Ls > 0.f) ? 1.f / Ls : 0.f;
#pragma unroll
  for (int j = 0; j < EPL; ++j) out[lane + 32 * j] = ElemT<T>::from_f(acc[j] * inv);
  if (lane == 0 && a.lse) {
    a.lse[(static_cast<int64_t>(b) * a.Lc + li) * a.Hq + gq] =
        (Ls > 0.f) ? (M + log2f(Ls)) * kLn2 : -INFINITY;
  }
}

template <typename T, int D, int QB>
void launch_partial_t(arbor_ctx *c, const AttnArgs &a, int S, int Lc) {
  constexpr int CH = kAttnChunk;
  constexpr int TG = 128 / (D / 2);
  const size_t smem = 2 * CH * D * sizeof(T) + CH * sizeof(int64_t) +
                      (QB * D + QB * CH + TG * QB * D + 2 * QB) * sizeof(float);
  static bool attr_set = false;
  if (!attr_set) {
    cudaFuncSetAttribute(attn_partial_kernel<T, D, QB>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         static_cast<int>(smem));
    attr_set = true;
  }
  dim3 grid(S, Lc, c->H);
  attn_partial_kernel<T, D, QB><<<grid, 128, smem, c->ms>>>(a);
}

template <typename T, int D>
void launch_partial_q(arbor_ctx *c, AttnArgs a, int S, int Lc, int max_q) {
  // queries per CTA batch: the smallest template ≥ min(max_q, 32) rounded to G multiples
  int qb;
  if (max_q <= 4) qb = 4;
  else if (max_q <= 8) qb = 8;
  else if (max_q <= 16) qb = 16;
  else qb = 32;
  a.lb_per = qb / a.G > 0 ? qb / a.G : 1;
  switch (qb) {
    case 4: launch_partial_t<T, D, 4>(c, a, S, Lc); break;
    case 8: launch_partial_t<T, D, 8>(c, a, S, Lc); break;
    case 16: launch_partial_t<T, D, 16>(c, a, S, Lc); break;
    default: launch_partial_t<T, D, 32>(c, a, S, Lc); break;
  }
}

}  // namespace

void launch_attn_partial(arbor_ctx *c, const PlanView &pv, int max_q, const void *q,
                         int layer_begin, int layer_count) {
  const int S = pv.S;
  if (S == 0) return;
  AttnArgs a{};
  a.pv = pv;
  a.g = PoolView{c->L, c->H, c->P, c->D, c->NP, c->max_pages_node, c->max_tokens};
  a.kpool = c->cfg.k_pool;
  a.vpool = c->cfg.v_pool;
  a.ptab = c->d.ptab;
  a.kcur = c->d.kcur;
  a.q = q;
  a.partials = c->d.partials;
  a.layer_begin = layer_begin;
  a.Lc = layer_count;
  a.Hq = c->Hq;
  a.G = c->G;
  a.scale_log2 = kLog2e / sqrtf(static_cast<float>(c->D));
  stage_begin(c, ARBOR_ST_ATTN, c->ms);
  if (c->esize == 2) {
    if (c->D == 128) launch_partial_q<__nv_bfloat16, 128>(c, a, S, layer_count, max_q);
    else launch_partial_q<__nv_bfloat16, 64>(c, a, S, layer_count, max_q);
  } else {
    if (c->D == 128) launch_partial_q<float, 128>(c, a, S, layer_count, max_q);
    else launch_partial_q<float, 64>(c, a, S, layer_count, max_q);
  }
  ARBOR_LAUNCHED(c);
  stage_end(c, ARBOR_ST_ATTN, c->ms);
}

void launch_attn_merge(arbor_ctx *c, const PlanView &pv, int layer_count, void *out,
                       float *lse) {
  const int nA = pv.nA;
  MergeArgs m{};
  m.pv = pv;
  m.partials = c->d.partials;
  m.out = out;
  m.lse = lse;
  m.Lc = layer_count;
  m.Hq = c->Hq;
  m.G = c->G;
  m.H = c->H;
  const int warps = nA * layer_count * c->Hq;
  const int blocks = (warps + 3) / 4;
  stage_begin(c, ARBOR_ST_ATTN_MERGE, c->ms);
  if (c->esize == 2) {
    if (c->D == 128) attn_merge_kernel<__nv_bfloat16, 128><<<blocks, 128, 0, c->ms>>>(m);
    else attn_merge_kernel<__nv_bfloat16, 64><<<blocks, 128, 0, c->ms>>>(m);
  } else {
    if (c->D == 128) attn_merge_kernel<float, 128><<<blocks, 128, 0, c->ms>>>(m);
    else attn_merge_kernel<float, 64><<<blocks, 128, 0, c->ms>>>(m);
  }
  ARBOR_LAUNCHED(c);
  stage_end(c, ARBOR_ST_ATTN_MERGE, c->ms);
}

}  // namespace arbor
