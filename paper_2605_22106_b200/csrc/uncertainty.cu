// uncertainty.cu — §8(f) f3: the boundary-time uncertainty feature of MSVE on the device.
//
// PAPER.md Eq. 1: p_i = softmax of the LM head's logits for the next token after
// block i closes; H_i = −Σ_{w∈𝒱} p_i(w) log p_i(w); u_i = 1 − H_i / log|𝒱| ∈ [0, 1].  The
// device evaluates the exact full-vocabulary sum (the paper's top-K + "other" bucket is an
// optional shortcut, whose entropy is never above the exact one).
//
// With a reference m: S = Σ e^{z−m}, T = Σ e^{z−m}(z − m), and H = log S − T/S.  Changing the
// reference to m' ≥ m rescales S' = e^{m−m'} S and T' = e^{m−m'} (T + (m − m') S), so each
// thread streams its slice once (8 logits per load batch, (m, S, T) in fp32), the CTA
// combines its threads' triples by shuffles, and the last CTA of a row (ticket) combines the
// CTAs' triples in fp64 and writes u.
// HBM-bound: one read of the logits (4 or 2 B per vocabulary entry).
#include <algorithm>

#include "common.cuh"

namespace arbor {
namespace {

constexpr int kUncThreads = 256;
constexpr int kUncPer = 8;           // logits per thread: loaded together, then absorbed
constexpr int kUncMaxSplit = 256;    // CTAs per row: ⌈vocab / (256·8)⌉, at most this

struct Triple {
  double m, S, T;
};

__device__ __forceinline__ Triple merge(Triple a, Triple b) {
  if (b.m == -INFINITY) return a;
  if (a.m == -INFINITY) return b;
  const double m = fmax(a.m, b.m);
  const double ra = exp(a.m - m), rb = exp(b.m - m);
  Triple t;
  t.m = m;
  t.S = ra * a.S + rb * b.S;
  t.T = ra * (a.T + (a.m - m) * a.S) + rb * (b.T + (b.m - m) * b.S);
  return t;
}

template <typename T>
__device__ __forceinline__ float to_f(T x);
template <>
__device__ __forceinline__ float to_f<float>(float x) { return x; }
template <>
__device__ __forceinline__ float to_f<__nv_bfloat16>(__nv_bfloat16 x) { return __bfloat162float(x); }

struct TripleF {
  float m, S, T;
};

__device__ __forceinline__ TripleF merge_f(TripleF a, TripleF b) {
  if (b.m == -INFINITY) return a;
  if (a.m == -INFINITY) return b;
  const float m = fmaxf(a.m, b.m);
  const float ra = expf(a.m - m), rb = expf(b.m - m);
  return TripleF{m, ra * a.S + rb * b.S, ra * (a.T + (a.m - m) * a.S) + rb * (b.T + (b.m - m) * b.S)};
}

template <typename T>
__global__ void __launch_bounds__(kUncThreads)
uncertainty_kernel(const T *__restrict__ logits, int vocab, Triple *__restrict__ part,
                   unsigned *__restrict__ ticket, float *__restrict__ u_out) {
  pdl_wait();
  pdl_trigger();
  const int row = blockIdx.y, split = blockIdx.x, nsplit = gridDim.x;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const T *z = logits + static_cast<int64_t>(row) * vocab;
  const int per = (vocab + nsplit - 1) / nsplit;
  const int lo = split * per, hi = min(vocab, lo + per);
  TripleF acc{-INFINITY, 0.f, 0.f};
  for (int i0 = lo + threadIdx.x; i0 < hi; i0 += kUncThreads * kUncPer) {
    float v[kUncPer];
    float m8 = -INFINITY;
#pragma unroll
    for (int j = 0; j < kUncPer; ++j) {       // all loads in flight before any use
      const int i = i0 + j * kUncThreads;
      v[j] = i < hi ? to_f(__ldg(z + i)) : -INFINITY;
    }
#pragma unroll
    for (int j = 0; j < kUncPer; ++j) m8 = fmaxf(m8, v[j]);
    if (m8 == -INFINITY) continue;            // all masked
    TripleF t{m8, 0.f, 0.f};
#pragma unroll
    for (int j = 0; j < kUncPer; ++j) {
      if (v[j] == -INFINITY) continue;        // a masked logit: p = 0
      const float d = v[j] - m8, e = expf(d);
      t.S += e;
      t.T = fmaf(e, d, t.T);
    }
    acc = merge_f(acc, t);
  }
  // warp, then CTA combine (fixed shuffle / slot order: deterministic)
#pragma unroll
  for (int o = 16; o; o >>= 1) {
    TripleF other{__shfl_xor_sync(0xffffffffu, acc.m, o), __shfl_xor_sync(0xffffffffu, acc.S, o),
                  __shfl_xor_sync(0xffffffffu, acc.T, o)};
    acc = lane & o ? merge_f(other, acc) : merge_f(acc, other);
  }
  __shared__ TripleF wred[kUncThreads / 32];
  if (lane == 0) wred[warp] = acc;
  __syncthreads();
  __shared__ bool last;
  if (threadIdx.x == 0) {
    TripleF c = wred[0];
    for (int w = 1; w < kUncThreads / 32; ++w) c = merge_f(c, wred[w]);
    part[row * nsplit + split] = Triple{static_cast<double>(c.m), static_cast<double>(c.S),
                                        static_cast<double>(c.T)};
    __threadfence();
    last = atomicAdd(&ticket[row], 1u) == static_cast<unsigned>(nsplit - 1);
  }
  __syncthreads();
  if (!last) return;
  // the row's last CTA: the CTAs' triples, loaded in parallel (L2), combined by a warp tree
  // in fp32 per 32 CTAs and in fp64 across those groups (fixed order: deterministic)
  __threadfence();
  if (warp != 0) return;
  Triple t{-INFINITY, 0.0, 0.0};
  for (int k0 = 0; k0 < nsplit; k0 += 32) {
    TripleF c{-INFINITY, 0.f, 0.f};
    if (k0 + lane < nsplit) {
      const Triple *p = part + row * nsplit + k0 + lane;
      c = TripleF{static_cast<float>(__ldcg(&p->m)), static_cast<float>(__ldcg(&p->S)),
                  static_cast<float>(__ldcg(&p->T))};
    }
#pragma unroll
    for (int o = 16; o; o >>= 1) {
      TripleF other{__shfl_xor_sync(0xffffffffu, c.m, o), __shfl_xor_sync(0xffffffffu, c.S, o),
                    __shfl_xor_sync(0xffffffffu, c.T, o)};
      c = lane & o ? merge_f(other, c) : merge_f(c, other);
    }
    t = merge(t, Triple{static_cast<double>(c.m), static_cast<double>(c.S), static_cast<double>(c.T)});
  }
  if (lane != 0) return;
  const double H = log(t.S) - t.T / t.S;
  const double u = 1.0 - H / log(static_cast<double>(vocab));
  u_out[row] = static_cast<float>(fmin(1.0, fmax(0.0, u)));
  ticket[row] = 0u;
}

}  // namespace

arbor_status launch_uncertainty(arbor_ctx *c, const void *logits, int dtype, int batch, int vocab,
                                float *u_out) {
  const int nsplit = std::min(kUncMaxSplit, std::max(1, (vocab + kUncThreads * kUncPer - 1) /
                                                            (kUncThreads * kUncPer)));
  const size_t need = static_cast<size_t>(batch) * kUncMaxSplit;
  if (need > c->unc_cap) {
    if (c->unc_part) cudaFree(c->unc_part);
    if (c->unc_ticket) cudaFree(c->unc_ticket);
    c->unc_part = nullptr;
    c->unc_ticket = nullptr;
    c->unc_cap = 0;
    if (cudaMalloc(&c->unc_part, need * sizeof(Triple)) != cudaSuccess ||
        cudaMalloc(&c->unc_ticket, static_cast<size_t>(batch) * sizeof(unsigned)) != cudaSuccess ||
        cudaMemsetAsync(c->unc_ticket, 0, static_cast<size_t>(batch) * sizeof(unsigned), c->ms) != cudaSuccess)
      return ARBOR_ERR_CUDA;
    c->unc_cap = need;
  }
  const dim3 grid(nsplit, batch);
  Triple *part = static_cast<Triple *>(c->unc_part);
  unsigned *tk = static_cast<unsigned *>(c->unc_ticket);
  cudaError_t e;
  if (dtype == ARBOR_BF16)
    e = launch_pdl(uncertainty_kernel<__nv_bfloat16>, grid, dim3(kUncThreads), 0, c->ms,
                   static_cast<const __nv_bfloat16 *>(logits), vocab, part, tk, u_out);
  else
    e = launch_pdl(uncertainty_kernel<float>, grid, dim3(kUncThreads), 0, c->ms,
                   static_cast<const float *>(logits), vocab, part, tk, u_out);
  ARBOR_LAUNCHED(c);
  return e == cudaSuccess ? ARBOR_OK : ARBOR_ERR_CUDA;
}

}  // namespace arbor
