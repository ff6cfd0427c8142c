// attn.cu — §8(a) a9: tree decode attention over the compacted ancestor-path pages.
//
// PAPER.md P:63 ("next-token decoding depends exclusively on the ancestor chain of the
// active leaf").  For every active leaf b, layer l and query head g
// (KV head h = g / G, Q24):  o = Σ_t softmax_t(q·k_t/√d) v_t over the retained slots of
// Path(ℓ_b), root→leaf; LSE = ln Σ_t exp(q·k_t/√d).
//
// B200 design (persistent, TMA-pipelined, CUDA-core math for few queries per KV head):
//  * Work item = (chunk of kAttnChunk slots of one node on the union of the active paths, a
//    subset of ≤ lmax leaves sharing it, layer, KV head).  A node shared by n active leaves
//    is read from HBM once for all of them (tree sharing) and once for all G query heads.
//  * One producer warp streams each item's K and V page-heads (≤ P rows × d, contiguous in
//    the pool) and the item's q rows into a 2-stage shared-memory ring with cp.async.bulk
//    (the TMA engine); completion is tracked by mbarrier transaction counts; 8 consumer
//    warps compute while the next item lands.  2 CTAs per SM, items strided across CTAs.
//  * QKᵀ: SL = d/16 lanes per token (16-element slices, log2(SL)-step shuffle reduce);
//    softmax statistics per query (warp per query); PV: lanes over 4-element column slices,
//    warps over token groups, smem reduction.  fp32 accumulation throughout.
//  * Each item emits split-softmax partials (Σ 2^{z−m} v, m, Σ 2^{z−m}) in the log2 domain
//    and its log2-domain logits z (consumed by the fused score pass, score.cu); a merge
//    kernel combines a leaf's partials in fixed root→leaf order (no float atomics).
#include <cfloat>

#include "tile.cuh"

namespace arbor {
namespace {

constexpr float kLn2 = 0.6931471805599453f;
constexpr float kLog2e = 1.4426950408889634f;
constexpr int kCh = kAttnChunk;      // slots per item
constexpr int kNst = 2;              // pipeline stages
constexpr int kConsumerWarps = 8;
constexpr int kConsumers = 32 * kConsumerWarps;
constexpr int kThreads = kConsumers + 32;

struct StreamArgs {
  PlanView pv;
  PoolView g;
  const void *kpool, *vpool;
  const int32_t *ptab, *kcur, *soff;
  const void *q;
  float *partials;   // [pair][Lc][H][G][D+2]
  float *zbuf;       // [pair][Lc][H][G][kCh] log2-domain logits
  int layer_begin, Lc, Hq, G, lmax, lb;   // lb: leaves per QB batch
  float scale_log2;  // log2(e)/sqrt(d)
};

struct StageHdr {
  int nt, li, h, pbase, cnt, lo, pad1, pad2;   // valid slots of the chunk: [lo, nt)
};

template <typename T>
__device__ __forceinline__ void load16(const T *p, float *f);
template <>
__device__ __forceinline__ void load16<__nv_bfloat16>(const __nv_bfloat16 *p, float *f) {
  const uint4 a = reinterpret_cast<const uint4 *>(p)[0];
  const uint4 b = reinterpret_cast<const uint4 *>(p)[1];
  ElemT<__nv_bfloat16>::cvt16(a, f);
  ElemT<__nv_bfloat16>::cvt16(b, f + 8);
}
template <>
__device__ __forceinline__ void load16<float>(const float *p, float *f) {
#pragma unroll
  for (int i = 0; i < 4; ++i) ElemT<float>::cvt16(reinterpret_cast<const uint4 *>(p)[i], f + 4 * i);
}

template <typename T>
__device__ __forceinline__ void load4(const T *p, float *f);
template <>
__device__ __forceinline__ void load4<__nv_bfloat16>(const __nv_bfloat16 *p, float *f) {
  const uint2 u = *reinterpret_cast<const uint2 *>(p);
  const float2 a = ElemT<__nv_bfloat16>::b2f(u.x), b = ElemT<__nv_bfloat16>::b2f(u.y);
  f[0] = a.x; f[1] = a.y; f[2] = b.x; f[3] = b.y;
}
template <>
__device__ __forceinline__ void load4<float>(const float *p, float *f) {
  const float4 v = *reinterpret_cast<const float4 *>(p);
  f[0] = v.x; f[1] = v.y; f[2] = v.z; f[3] = v.w;
}

template <typename T, int D, int QB>
__global__ void __launch_bounds__(kThreads, 2)
attn_stream_kernel(StreamArgs a) {
  constexpr int SL = D / 16;                // lanes per token in QKᵀ
  constexpr int TPP = kConsumers / SL;      // tokens per QKᵀ pass
  constexpr int S4 = D / 4;                 // 4-element column slices in PV
  constexpr int RPW = 32 / S4;              // rows per warp in PV
  constexpr int TG = kConsumerWarps * RPW;  // token groups in PV
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int G = a.G;
  const int qcap = a.lmax * G;              // q rows staged per item
  const int64_t stage_elems = static_cast<int64_t>(2 * kCh * D + qcap * D);
  extern __shared__ __align__(128) unsigned char sm[];
  T *stage0 = reinterpret_cast<T *>(sm);
  float *zs = reinterpret_cast<float *>(stage0 + kNst * stage_elems);   // [kCh][QB]
  float *red = zs + kCh * QB;                                           // [TG][QB][D]
  float *mls = red + TG * QB * D;                                       // m2[QB], l[QB]
  StageHdr *hdr = reinterpret_cast<StageHdr *>(mls + 2 * QB);
  uint64_t *full = reinterpret_cast<uint64_t *>(hdr + kNst);
  uint64_t *empty = full + kNst;
  if (tid == 0) {
    for (int s = 0; s < kNst; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], kConsumerWarps);
    }
    mbar_fence_init();
  }
  __syncthreads();
  const int total = a.pv.I * a.Lc * a.g.H;
  const int rb = D * static_cast<int>(sizeof(T));
  const T *q = static_cast<const T *>(a.q);
  if (warp == 0) {
    // ------------------------------------------------------------- producer (TMA)
    // The whole warp fetches an item's metadata (one int4 record, then k_cur, page ids and
    // pair ids in parallel) one item ahead; lane i issues the bulk copies of page i.
    const T *kpool = static_cast<const T *>(a.kpool);
    const T *vpool = static_cast<const T *>(a.vpool);
    const int lgP = 31 - __clz(a.g.P);
    const int pages_per_item = a.g.P >= kCh ? 1 : kCh / a.g.P;
    struct Meta { int4 rec; int kc, so, page, b; };
    auto fetch = [&](int it, Meta &m) {
      if (it >= total) return;
      const int item = it / (a.g.H * a.Lc);
      m.rec = a.pv.it_rec[item];
      m.kc = a.kcur[m.rec.x];
      m.so = a.soff[m.rec.x];
      m.page = lane < pages_per_item
                   ? a.ptab[static_cast<int64_t>(m.rec.x) * a.g.MPN + (m.rec.y >> lgP) + lane] : 0;
      m.b = lane < m.rec.w ? a.pv.pair_b[m.rec.z + lane] : 0;
    };
    Meta cur{}, nxt{};
    fetch(blockIdx.x, cur);
    int k = 0;
    for (int it = blockIdx.x; it < total; it += gridDim.x, ++k) {
      fetch(it + gridDim.x, nxt);                  // loads in flight during the wait below
      const int st = k % kNst;
      const uint32_t ph = (k / kNst) & 1u;
      const int h = it % a.g.H;
      const int li = (it / a.g.H) % a.Lc;
      const int node = cur.rec.x, c0 = cur.rec.y, pbase = cur.rec.z, cnt = cur.rec.w;
      (void)node;
      // rows [0, hi) of the chunk are loaded, those below lo (stale pages before soff,
      // DESIGN.md Q23*) masked
      const int span = chunk_span(cur.so, cur.kc, c0, kCh);
      const int nt = span_hi(span), lo = span_lo(span);
      mbar_wait(&empty[st], ph ^ 1u);
      T *Ks = stage0 + st * stage_elems;
      T *Vs = Ks + kCh * D;
      T *Qs = Vs + kCh * D;
      if (lane == 0) {
        hdr[st] = StageHdr{nt, li, h, pbase, cnt, lo, 0, 0};
        mbar_arrive_expect_tx(&full[st], static_cast<uint32_t>((2 * nt + cnt * G) * rb));
      }
      __syncwarp();
      const int l = a.layer_begin + li;
      if (lane < pages_per_item) {
        const int off = a.g.P >= kCh ? (c0 & (a.g.P - 1)) : 0;
        const int s0 = lane * (a.g.P >= kCh ? 0 : a.g.P);
        const int rows = min(a.g.P >= kCh ? kCh : a.g.P, nt - s0);
        if (rows > 0) {
          const int64_t row = pool_row(a.g, l, cur.page, h, off);
          bulk_g2s(Ks + s0 * D, kpool + row * D, rows * rb, &full[st]);
          bulk_g2s(Vs + s0 * D, vpool + row * D, rows * rb, &full[st]);
        }
      }
      if (lane < cnt)
        bulk_g2s(Qs + lane * G * D,
                 q + ((static_cast<int64_t>(cur.b) * a.Lc + li) * a.Hq + h * G) * D, G * rb,
                 &full[st]);
      cur = nxt;
    }
    return;
  }
  // --------------------------------------------------------------- consumers
  const int ct = tid - 32;
  int k = 0;
  for (int it = blockIdx.x; it < total; it += gridDim.x, ++k) {
    const int st = k % kNst;
    const uint32_t ph = (k / kNst) & 1u;
    mbar_wait(&full[st], ph);
    const StageHdr hd = hdr[st];
    const int nt = hd.nt, lo = hd.lo, li = hd.li, h = hd.h, cnt = hd.cnt, pbase = hd.pbase;
    const T *Ks = stage0 + st * stage_elems;
    const T *Vs = Ks + kCh * D;
    const T *Qs = Vs + kCh * D;
    for (int b0 = 0; b0 < cnt; b0 += a.lb) {
      const int nb = min(a.lb, cnt - b0);
      const int nq = nb * G;
      // ---- phase 1: z[t][qi] = log2(e)/√d · q·k_t, in groups of 4 queries
      {
        const int sl = ct % SL, tt = ct / SL;
        for (int q0 = 0; q0 < nq; q0 += 4) {
          float qf[4][16];
#pragma unroll
          for (int qi = 0; qi < 4; ++qi) {
            if (q0 + qi < nq) {
              load16<T>(Qs + (b0 * G + q0 + qi) * D + sl * 16, qf[qi]);
            } else {
#pragma unroll
              for (int e = 0; e < 16; ++e) qf[qi][e] = 0.f;
            }
          }
          for (int t0 = 0; t0 < kCh; t0 += TPP) {
            const int t = t0 + tt;
            float dot[4] = {0.f, 0.f, 0.f, 0.f};
            if (t >= lo && t < nt) {
              float kf[16];
              load16<T>(Ks + t * D + sl * 16, kf);
#pragma unroll
              for (int qi = 0; qi < 4; ++qi) {
                float acc = 0.f;
#pragma unroll
                for (int e = 0; e < 16; ++e) acc = fmaf(kf[e], qf[qi][e], acc);
                dot[qi] = acc;
              }
            }
#pragma unroll
            for (int qi = 0; qi < 4; ++qi) {
#pragma unroll
              for (int o = SL / 2; o; o >>= 1) dot[qi] += __shfl_xor_sync(0xffffffffu, dot[qi], o);
            }
            if (sl == 0) {
#pragma unroll
              for (int qi = 0; qi < 4; ++qi)
                if (q0 + qi < QB)
                  zs[t * QB + q0 + qi] = (t >= lo && t < nt && q0 + qi < nq) ? dot[qi] * a.scale_log2 : -INFINITY;
            }
          }
        }
      }
      named_bar_sync(1, kConsumers);
      // logits for the fused score pass: zbuf[pair][li][h][g][t]
      for (int idx = ct; idx < nq * kCh; idx += kConsumers) {
        const int qi = idx / kCh, t = idx - qi * kCh;
        const int bi = qi / G, g = qi - bi * G;
        a.zbuf[((((static_cast<int64_t>(pbase + b0 + bi)) * a.Lc + li) * a.g.H + h) * G + g) * kCh + t] =
            zs[t * QB + qi];
      }
      // ---- phase 2: per-query max and exp-sum over the chunk (warp per query)
      for (int qi = warp - 1; qi < nq; qi += kConsumerWarps) {
        float v[kCh / 32];
        float m = -INFINITY;
#pragma unroll
        for (int j = 0; j < kCh / 32; ++j) {
          v[j] = zs[(lane + 32 * j) * QB + qi];
          m = fmaxf(m, v[j]);
        }
#pragma unroll
        for (int o = 16; o; o >>= 1) m = fmaxf(m, __shfl_xor_sync(0xffffffffu, m, o));
        float sum = 0.f;
#pragma unroll
        for (int j = 0; j < kCh / 32; ++j) {
          const float p = (v[j] == -INFINITY) ? 0.f : exp2f(v[j] - m);
          zs[(lane + 32 * j) * QB + qi] = p;
          sum += p;
        }
#pragma unroll
        for (int o = 16; o; o >>= 1) sum += __shfl_xor_sync(0xffffffffu, sum, o);
        if (lane == 0) {
          mls[qi] = m;
          mls[QB + qi] = sum;
        }
      }
      named_bar_sync(1, kConsumers);
      // ---- phase 3: o = Σ_t p_t v_t; lanes over 4-element column slices, warps over tokens
      {
        const int e4 = lane % S4, tg = (warp - 1) * RPW + lane / S4;
        float acc[QB][4];
#pragma unroll
        for (int qi = 0; qi < QB; ++qi) acc[qi][0] = acc[qi][1] = acc[qi][2] = acc[qi][3] = 0.f;
        for (int t = lo + tg; t < nt; t += TG) {   // rows below lo: not the node's (Q23*)
          float vf[4];
          load4<T>(Vs + t * D + e4 * 4, vf);
          float p[QB];
#pragma unroll
          for (int qi = 0; qi < QB; qi += 4) {
            const float4 pp = *reinterpret_cast<const float4 *>(zs + t * QB + qi);
            p[qi] = pp.x; p[qi + 1] = pp.y; p[qi + 2] = pp.z; p[qi + 3] = pp.w;
          }
#pragma unroll
          for (int qi = 0; qi < QB; ++qi)
#pragma unroll
            for (int e = 0; e < 4; ++e) acc[qi][e] = fmaf(p[qi], vf[e], acc[qi][e]);
        }
#pragma unroll
        for (int qi = 0; qi < QB; ++qi)
          if (qi < nq)
            *reinterpret_cast<float4 *>(red + (tg * QB + qi) * D + e4 * 4) =
                make_float4(acc[qi][0], acc[qi][1], acc[qi][2], acc[qi][3]);
      }
      named_bar_sync(1, kConsumers);
      if (b0 + a.lb >= cnt && lane == 0) mbar_arrive(&empty[st]);   // stage no longer read
      for (int idx = ct; idx < nq * (D + 2); idx += kConsumers) {
        const int qi = idx / (D + 2), e = idx - qi * (D + 2);
        const int bi = qi / G, g = qi - bi * G;
        float val;
        if (e < D) {
          val = 0.f;
#pragma unroll 8
          for (int j = 0; j < TG; ++j) val += red[(j * QB + qi) * D + e];
        } else {
          val = mls[(e - D) * QB + qi];
        }
        a.partials[((((static_cast<int64_t>(pbase + b0 + bi)) * a.Lc + li) * a.g.H + h) * G + g) *
                       (D + 2) + e] = val;
      }
      named_bar_sync(1, kConsumers);
    }
    if (cnt == 0 && lane == 0) mbar_arrive(&empty[st]);
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
  pdl_wait();
  pdl_trigger();
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
void launch_stream_t(arbor_ctx *c, StreamArgs a) {
  constexpr int S4 = D / 4, RPW = 32 / S4, TG = kConsumerWarps * RPW;
  const size_t stage = (2 * kCh * D + static_cast<size_t>(a.lmax) * a.G * D) * sizeof(T);
  const size_t smem = kNst * stage + (kCh * QB + TG * QB * D + 2 * QB) * sizeof(float) +
                      kNst * sizeof(StageHdr) + 2 * kNst * sizeof(uint64_t) + 16;
  static size_t attr = 0;
  if (smem > attr) {
    cudaFuncSetAttribute(attn_stream_kernel<T, D, QB>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         static_cast<int>(smem));
    attr = smem;
  }
  int sms = 148;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  int per_sm = 0;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, attn_stream_kernel<T, D, QB>, kThreads, smem);
  const int total = a.pv.I * a.Lc * a.g.H;
  int grid = sms * (per_sm > 0 ? per_sm : 1);
  if (grid > total) grid = total;
  attn_stream_kernel<T, D, QB><<<grid, kThreads, smem, c->ms>>>(a);
}

template <typename T, int D>
void launch_stream_q(arbor_ctx *c, StreamArgs a) {
  if (a.G <= 4) {
    a.lb = 4 / a.G;
    launch_stream_t<T, D, 4>(c, a);
  } else {
    a.lb = 8 / a.G;
    launch_stream_t<T, D, 8>(c, a);
  }
}

}  // namespace

bool launch_attn_partial(arbor_ctx *c, const PlanView &pv, const void *q, int layer_begin,
                         int layer_count, int max_cnt, void *out, float *lse) {
  if (pv.I == 0) return false;
  stage_begin(c, ARBOR_ST_ATTN, c->ms);
  if (launch_attn_tc(c, pv, q, layer_begin, layer_count, max_cnt, out, lse)) {   // attn_tc.cu
    ARBOR_LAUNCHED(c);
    stage_end(c, ARBOR_ST_ATTN, c->ms);
    return false;   // partials only: merged by attn_merge_kernel
  }
  StreamArgs a{};
  a.pv = pv;
  a.g = PoolView{c->L, c->H, c->P, c->D, c->NP, c->max_pages_node, c->max_tokens};
  a.kpool = c->cfg.k_pool;
  a.vpool = c->cfg.v_pool;
  a.ptab = c->d.ptab;
  a.kcur = c->d.kcur;
  a.soff = c->d.soff;
  a.q = q;
  a.partials = c->d.partials;
  a.zbuf = c->d.zbuf;
  a.layer_begin = layer_begin;
  a.Lc = layer_count;
  a.Hq = c->Hq;
  a.G = c->G;
  a.lmax = kLeavesPerItem;
  a.scale_log2 = kLog2e / sqrtf(static_cast<float>(c->D));
  if (c->esize == 2) {
    if (c->D == 128) launch_stream_q<__nv_bfloat16, 128>(c, a);
    else launch_stream_q<__nv_bfloat16, 64>(c, a);
  } else {
    if (c->D == 128) launch_stream_q<float, 128>(c, a);
    else launch_stream_q<float, 64>(c, a);
  }
  ARBOR_LAUNCHED(c);
  stage_end(c, ARBOR_ST_ATTN, c->ms);
  return false;
}

void launch_attn_merge(arbor_ctx *c, const PlanView &pv, int layer_count, void *out, float *lse) {
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
    if (c->D == 128) launch_pdl(attn_merge_kernel<__nv_bfloat16, 128>, dim3(blocks), dim3(128), 0, c->ms, m);
    else launch_pdl(attn_merge_kernel<__nv_bfloat16, 64>, dim3(blocks), dim3(128), 0, c->ms, m);
  } else {
    if (c->D == 128) launch_pdl(attn_merge_kernel<float, 128>, dim3(blocks), dim3(128), 0, c->ms, m);
    else launch_pdl(attn_merge_kernel<float, 64>, dim3(blocks), dim3(128), 0, c->ms, m);
  }
  ARBOR_LAUNCHED(c);
  stage_end(c, ARBOR_ST_ATTN_MERGE, c->ms);
}

}  // namespace arbor
