// uncertainty.cu — §8(f) f3: the boundary-time uncertainty feature of MSVE on the device.
//
// PAPER.md Eq. 1: p_i = softmax of the LM head's logits for the next token after
// block i closes; H_i = −Σ_{w∈𝒱} p_i(w) log p_i(w); u_i = 1 − H_i / log|𝒱| ∈ [0, 1].  The
// device evaluates the exact full-vocabulary sum (the paper's top-K + "other" bucket is an
// optional shortcut, whose entropy is never above the exact one).
//
// With a reference m: S = Σ e^{z−m}, T = Σ e^{z−m}(z − m), and H = log S − T/S.  Changing the
// reference to m' ≥ m rescales S' = e^{m−m'} S and T' = e^{m−m'} (T + (m − m') S), so each
// thread streams its slice once (online m, S, T in fp32), CTAs combine their threads' triples
// in fp64, and the last CTA of a row (ticket) combines the CTAs' triples and writes u.
// HBM-bound: one read of the logits (4 or 2 B per vocabulary entry).
#include "common.cuh"

namespace arbor {
namespace {

constexpr int kUncThreads = 256;
constexpr int kUncSplit = 16;        // CTAs per row (grid = batch × kUncSplit)

struct Triple {
  double m, S, T;
};

__device__ __forceinline__ void absorb(float &m, float &S, float &T, float z) {
  if (z == -INFINITY) return;               // a masked logit: p = 0 contributes nothing
  if (z > m) {
    const float r = m == -INFINITY ? 0.f : expf(m - z);
    T = r * (T + (m == -INFINITY ? 0.f : (m - z)) * S);
    S = r * S;
    m = z;
  }
  const float e = expf(z - m);
  S += e;
  T += e * (z - m);
}

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

template <typename T>
__global__ void __launch_bounds__(kUncThreads)
uncertainty_kernel(const T *__restrict__ logits, int vocab, Triple *__restrict__ part,
                   unsigned *__restrict__ ticket, float *__restrict__ u_out) {
  pdl_wait();
  pdl_trigger();
  const int row = blockIdx.y, split = blockIdx.x;
  const T *z = logits + static_cast<int64_t>(row) * vocab;
  const int per = (vocab + kUncSplit - 1) / kUncSplit;
  const int lo = split * per, hi = min(vocab, lo + per);
  float m = -INFINITY, S = 0.f, Tt = 0.f;
  for (int i = lo + threadIdx.x; i < hi; i += kUncThreads) absorb(m, S, Tt, to_f(__ldg(z + i)));
  // block combine (fp64) through shared memory
  __shared__ Triple red[kUncThreads];
  red[threadIdx.x] = Triple{static_cast<double>(m), static_cast<double>(S), static_cast<double>(Tt)};
  __syncthreads();
  for (int s = kUncThreads / 2; s > 0; s >>= 1) {
    if (threadIdx.x < s) red[threadIdx.x] = merge(red[threadIdx.x], red[threadIdx.x + s]);
    __syncthreads();
  }
  __shared__ bool last;
  if (threadIdx.x == 0) {
    part[row * kUncSplit + split] = red[0];
    __threadfence();
    last = atomicAdd(&ticket[row], 1u) == kUncSplit - 1;
  }
  __syncthreads();
  if (!last || threadIdx.x != 0) return;
  __threadfence();
  Triple t{-INFINITY, 0.0, 0.0};
  for (int k = 0; k < kUncSplit; ++k) {   // fixed order: deterministic
    const volatile Triple *p = part + row * kUncSplit + k;
    t = merge(t, Triple{p->m, p->S, p->T});
  }
  const double H = log(t.S) - t.T / t.S;
  const double u = 1.0 - H / log(static_cast<double>(vocab));
  u_out[row] = static_cast<float>(fmin(1.0, fmax(0.0, u)));
  ticket[row] = 0u;
}

}  // namespace

arbor_status launch_uncertainty(arbor_ctx *c, const void *logits, int dtype, int batch, int vocab,
                                float *u_out) {
  const size_t need = static_cast<size_t>(batch) * kUncSplit;
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
  const dim3 grid(kUncSplit, batch);
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
