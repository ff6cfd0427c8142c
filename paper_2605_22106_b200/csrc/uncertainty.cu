// uncertainty.cu — §8(f) f3: the boundary-time uncertainty feature of MSVE on the device.
//
// PAPER.md Eq. 1: p_i = softmax of the LM head's logits for the next token after
// block i closes; H_i = −Σ_{w∈𝒱} p_i(w) log p_i(w); u_i = 1 − H_i / log|𝒱| ∈ [0, 1].  The
// device evaluates the exact full-vocabulary sum (the paper's top-K + "other" bucket is an
// optional shortcut, whose entropy is never above the exact one).
//
// With a reference m: S = Σ e^{z−m}, T = Σ e^{z−m}(z − m), and H = log S − T/S.  Changing the
// reference to m' ≥ m rescales S' = e^{m−m'} S and T' = e^{m−m'} (T + (m − m') S), so each
// thread streams its slice once (16-byte vector loads, four in flight, (m, S, T) in fp32), the CTA
// combines its threads' triples by shuffles, and the last CTA of a row (ticket) combines the
// CTAs' triples in fp64 and writes u.
// HBM-bound: one read of the logits (4 or 2 B per vocabulary entry).
#include <algorithm>
#include <cmath>

#include "common.cuh"

namespace arbor {
namespace {

constexpr int kUncThreads = 256;
constexpr int kUncVecs = 4;          // 16-byte vectors per thread in flight per step
constexpr int kUncMaxSplit = 256;    // CTAs per row (at most)
#ifndef ARBOR_UNC_PER_CTA
#define ARBOR_UNC_PER_CTA 16384
#endif
constexpr int kUncPerCta = ARBOR_UNC_PER_CTA;   // logits per CTA (about)

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

// 16-byte vector of logits and its element count
template <typename T> struct UncVec;
template <> struct UncVec<float> {
  static constexpr int N = 4;
  __device__ __forceinline__ static void load(const float *p, float (&v)[4]) {
    const float4 q = __ldg(reinterpret_cast<const float4 *>(p));
    v[0] = q.x; v[1] = q.y; v[2] = q.z; v[3] = q.w;
  }
};
template <> struct UncVec<__nv_bfloat16> {
  static constexpr int N = 8;
  __device__ __forceinline__ static void load(const __nv_bfloat16 *p, float (&v)[8]) {
    const uint4 q = __ldg(reinterpret_cast<const uint4 *>(p));
    const uint32_t w[4] = {q.x, q.y, q.z, q.w};
#pragma unroll
    for (int k = 0; k < 4; ++k) {   // bf16 → f32 is a 16-bit shift: exact
      v[2 * k] = __uint_as_float(w[k] << 16);
      v[2 * k + 1] = __uint_as_float(w[k] & 0xffff0000u);
    }
  }
};

// absorb n logits (−inf: masked, p = 0) into the running triple, one rescale per call
template <int NV>
__device__ __forceinline__ void absorb(TripleF &acc, const float (&v)[NV]) {
  float mx = -INFINITY;
#pragma unroll
  for (int j = 0; j < NV; ++j) mx = fmaxf(mx, v[j]);
  if (mx == -INFINITY) return;
  TripleF t{mx, 0.f, 0.f};
#pragma unroll
  for (int j = 0; j < NV; ++j) {
    const float d = v[j] - mx, e = v[j] == -INFINITY ? 0.f : expf(d);
    t.S += e;
    t.T = fmaf(e, v[j] == -INFINITY ? 0.f : d, t.T);
  }
  acc = merge_f(acc, t);
}

// Row `row`, split `split` of `nsplit`: the row's 16-byte-aligned body is cut into nsplit
// ranges of whole vectors (kUncVecs vectors per thread in flight per step); the unaligned head
// (< one vector) goes to split 0 and the tail to the last split, element by element.
template <typename T>
__global__ void __launch_bounds__(kUncThreads)
uncertainty_kernel(const T *__restrict__ logits, int vocab, Triple *__restrict__ part,
                   unsigned *__restrict__ ticket, float *__restrict__ u_out) {
  pdl_wait();
  pdl_trigger();
  constexpr int NV = UncVec<T>::N;
  const int row = blockIdx.y, split = blockIdx.x, nsplit = gridDim.x;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const T *z = logits + static_cast<int64_t>(row) * vocab;
  const int head = min(vocab, static_cast<int>(((16 - (reinterpret_cast<uintptr_t>(z) & 15)) & 15) / sizeof(T)));
  const int nvec = (vocab - head) / NV;                  // whole vectors of the body
  const int tail0 = head + nvec * NV;                    // first element of the tail
  const int vper = (nvec + nsplit - 1) / nsplit;
  const int v_lo = min(nvec, split * vper), v_hi = min(nvec, v_lo + vper);
  const T *body = z + head;
  TripleF acc{-INFINITY, 0.f, 0.f};
  for (int v0 = v_lo + threadIdx.x; v0 < v_hi; v0 += kUncThreads * kUncVecs) {
    float v[kUncVecs][NV];
#pragma unroll
    for (int k = 0; k < kUncVecs; ++k) {      // every load in flight before any use
      const int vi = v0 + k * kUncThreads;
      if (vi < v_hi) {
        UncVec<T>::load(body + static_cast<int64_t>(vi) * NV, v[k]);
      } else {
#pragma unroll
        for (int j = 0; j < NV; ++j) v[k][j] = -INFINITY;
      }
    }
#pragma unroll
    for (int k = 0; k < kUncVecs; ++k) absorb<NV>(acc, v[k]);
  }
  // the unaligned head (split 0) and tail (last split): one element per thread
  {
    const bool first = split == 0, lastsplit = split == nsplit - 1;
    float e1[1] = {-INFINITY};
    if (first && static_cast<int>(threadIdx.x) < head) e1[0] = to_f(z[threadIdx.x]);
    else if (lastsplit && static_cast<int>(threadIdx.x) < vocab - tail0) e1[0] = to_f(z[tail0 + threadIdx.x]);
    absorb<1>(acc, e1);
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
  // logits per CTA: about half a wave of CTAs in total, within [4096, kUncPerCta] (measured:
  // 4096 best for one row, 16384 for 64 rows of a 128k vocabulary)
  const int64_t want = static_cast<int64_t>(vocab) * batch / 512;
  const int per = static_cast<int>(std::min<int64_t>(kUncPerCta, std::max<int64_t>(4096, want)));
  const int nsplit = std::min(kUncMaxSplit, std::max(1, (vocab + per - 1) / per));
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


// ---------------------------------------------------------------- f3: MSVE θ calibration
// Full-batch gradient descent of L(θ) = mean_i (σ(θᵀx_i) − y_i)², x_i = (1, v_i, u_i, a_i),
// with loss-nonincrease backoff (a step that raises the loss halves the rate and retries, at
// most 20 halvings, the reduced rate is kept) — oracle/calibrate.py.  One CTA
// runs every epoch: thread t sums examples t, t + 256, … in fp64, then a fixed-order tree
// reduction in shared memory (deterministic); z = θ₀ + θ_v v + θ_u u + θ_a a left to right.
namespace {
constexpr int kFitThreads = 256;

__device__ __forceinline__ double fit_sigma(const double *th, float v, float u, float a) {
  double z = __dadd_rn(th[0], __dmul_rn(th[1], static_cast<double>(v)));
  z = __dadd_rn(z, __dmul_rn(th[2], static_cast<double>(u)));
  z = __dadd_rn(z, __dmul_rn(th[3], static_cast<double>(a)));
  return 1.0 / (1.0 + exp(-z));
}

// block sum of per-thread values (fixed tree order); every thread gets the result
template <int W>
__device__ __forceinline__ void block_sum_vec(double (&v)[W], double (*red)[kFitThreads]) {
  for (int k = 0; k < W; ++k) red[k][threadIdx.x] = v[k];
  __syncthreads();
  for (int off = kFitThreads / 2; off > 0; off >>= 1) {
    if (threadIdx.x < off)
      for (int k = 0; k < W; ++k) red[k][threadIdx.x] += red[k][threadIdx.x + off];
    __syncthreads();
  }
  for (int k = 0; k < W; ++k) v[k] = red[k][0];
  __syncthreads();
}

__global__ void __launch_bounds__(kFitThreads)
fit_theta_kernel(const float *__restrict__ phi, const float *__restrict__ y, int n, int epochs,
                 double lr, double *theta_io, double *loss_io) {
  __shared__ double red[4][kFitThreads];
  __shared__ double th[4], cand[4];
  if (threadIdx.x < 4) th[threadIdx.x] = theta_io[threadIdx.x];
  __syncthreads();
  const double inv_n = 1.0 / static_cast<double>(n);
  auto loss_of = [&](const double *t) {
    double acc[1] = {0.0};
    for (int i = threadIdx.x; i < n; i += kFitThreads) {
      const double d = fit_sigma(t, phi[3 * i], phi[3 * i + 1], phi[3 * i + 2]) - static_cast<double>(y[i]);
      acc[0] += d * d;
    }
    block_sum_vec<1>(acc, red);
    return acc[0] * inv_n;
  };
  double cur = loss_of(th);
  const double first = cur;
  for (int ep = 0; ep < epochs; ++ep) {
    double g[4] = {0.0, 0.0, 0.0, 0.0};
    for (int i = threadIdx.x; i < n; i += kFitThreads) {
      const float v = phi[3 * i], u = phi[3 * i + 1], a = phi[3 * i + 2];
      const double s = fit_sigma(th, v, u, a);
      const double c = 2.0 * (s - static_cast<double>(y[i])) * s * (1.0 - s);
      g[0] += c;
      g[1] += c * v;
      g[2] += c * u;
      g[3] += c * a;
    }
    block_sum_vec<4>(g, red);
    for (int k = 0; k < 4; ++k) g[k] *= inv_n;
    double step = lr, lc = 0.0;
    bool ok = false;
    for (int tr = 0; tr < 21; ++tr) {
      if (threadIdx.x < 4) cand[threadIdx.x] = th[threadIdx.x] - step * g[threadIdx.x];
      __syncthreads();
      lc = loss_of(cand);
      if (lc <= cur) { ok = true; break; }
      step *= 0.5;
    }
    if (!ok) break;
    if (threadIdx.x < 4) th[threadIdx.x] = cand[threadIdx.x];
    __syncthreads();
    cur = lc;
    lr = step;
  }
  if (threadIdx.x < 4) theta_io[threadIdx.x] = th[threadIdx.x];
  if (threadIdx.x == 0) { loss_io[0] = first; loss_io[1] = cur; }
}
}  // namespace

}  // namespace arbor

extern "C" arbor_status arbor_fit_theta(const float *phi, const float *target, int32_t n,
                                        int32_t epochs, double lr, double *theta,
                                        double *loss_out) {
  if (!phi || !target || !theta || n < 1 || epochs < 0 || !(lr > 0.0)) return ARBOR_ERR_INVALID_ARG;
  for (int k = 0; k < 4; ++k) if (!std::isfinite(theta[k])) return ARBOR_ERR_INVALID_ARG;
  double *d = nullptr;
  if (cudaMalloc(&d, 6 * sizeof(double)) != cudaSuccess) return ARBOR_ERR_CUDA;
  arbor_status st = ARBOR_OK;
  double h[6] = {theta[0], theta[1], theta[2], theta[3], 0.0, 0.0};
  if (cudaMemcpy(d, h, 4 * sizeof(double), cudaMemcpyHostToDevice) != cudaSuccess) st = ARBOR_ERR_CUDA;
  if (st == ARBOR_OK) {
    arbor::fit_theta_kernel<<<1, arbor::kFitThreads>>>(phi, target, n, epochs, lr, d, d + 4);
    if (cudaGetLastError() != cudaSuccess || cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost) != cudaSuccess)
      st = ARBOR_ERR_CUDA;
  }
  cudaFree(d);
  if (st != ARBOR_OK) return st;
  for (int k = 0; k < 4; ++k) theta[k] = h[k];
  if (loss_out) { loss_out[0] = h[4]; loss_out[1] = h[5]; }
  return ARBOR_OK;
}
