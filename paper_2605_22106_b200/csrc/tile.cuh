// tile.cuh — paged K/V tile staging shared by the attention and score kernels.
#pragma once
#ifdef ARBOR_MBAR_WATCHDOG
#include <cstdio>   // the debug watchdog's report (mbar_wait below)
#endif
#include "common.cuh"

namespace arbor {

template <typename T> struct ElemT;
template <> struct ElemT<float> {
  static constexpr int kPer16 = 4;
  __device__ __forceinline__ static void cvt16(const uint4 &r, float *f) {
    f[0] = __uint_as_float(r.x); f[1] = __uint_as_float(r.y);
    f[2] = __uint_as_float(r.z); f[3] = __uint_as_float(r.w);
  }
  __device__ __forceinline__ static float2 ld2(const float *p) {
    return *reinterpret_cast<const float2 *>(p);
  }
  __device__ __forceinline__ static float to_f(float x) { return x; }
  __device__ __forceinline__ static float from_f(float x) { return x; }
};
template <> struct ElemT<__nv_bfloat16> {
  static constexpr int kPer16 = 8;
  __device__ __forceinline__ static float2 b2f(uint32_t u) {
    // bf16 → f32 is a 16-bit shift: exact
    return make_float2(__uint_as_float(u << 16), __uint_as_float(u & 0xffff0000u));
  }
  __device__ __forceinline__ static void cvt16(const uint4 &r, float *f) {
    float2 a = b2f(r.x), b = b2f(r.y), c = b2f(r.z), d = b2f(r.w);
    f[0] = a.x; f[1] = a.y; f[2] = b.x; f[3] = b.y; f[4] = c.x; f[5] = c.y; f[6] = d.x; f[7] = d.y;
  }
  __device__ __forceinline__ static float2 ld2(const __nv_bfloat16 *p) {
    return b2f(*reinterpret_cast<const uint32_t *>(p));
  }
  __device__ __forceinline__ static float to_f(__nv_bfloat16 x) { return __bfloat162float(x); }
  __device__ __forceinline__ static __nv_bfloat16 from_f(float x) { return __float2bfloat16_rn(x); }
};

__device__ __forceinline__ void cp_async16(void *smem, const void *gmem) {
  const uint32_t s = static_cast<uint32_t>(__cvta_generic_to_shared(smem));
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(s), "l"(gmem));
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::); }
__device__ __forceinline__ void cp_async_wait_all() {
  asm volatile("cp.async.wait_all;\n" ::: "memory");
}

// Row index of (layer l, page, kv head h, slot offset) in a [L][NP][H][P] pool.
__device__ __forceinline__ int64_t pool_row(const PoolView &g, int l, int page, int h, int off) {
  return ((static_cast<int64_t>(l) * g.NP + page) * g.H + h) * g.P + off;
}


// Dot products of the thread's K row (row t of the swizzled tile) with nq ≤ QB query rows
// held in smem as f32 [QB][D]; acc[qi] = q_qi · k_t.
template <typename T, int D, int QB>
__device__ __forceinline__ void row_dots(const T *Ks, const float *qs, int t, int nq,
                                         float (&acc)[QB]) {
  constexpr int EPV = ElemT<T>::kPer16;
  constexpr int CPR = D / EPV;
#pragma unroll
  for (int qi = 0; qi < QB; ++qi) acc[qi] = 0.f;
#pragma unroll 4
  for (int cc = 0; cc < CPR; ++cc) {
    const uint4 raw = *reinterpret_cast<const uint4 *>(
        reinterpret_cast<const char *>(Ks + t * D) + ((cc ^ (t & 7)) * 16));
    float kf[EPV];
    ElemT<T>::cvt16(raw, kf);
#pragma unroll
    for (int qi = 0; qi < QB; ++qi) {
      if (qi < nq) {
        const float4 *qp = reinterpret_cast<const float4 *>(qs + qi * D + cc * EPV);
#pragma unroll
        for (int v4 = 0; v4 < EPV / 4; ++v4) {
          const float4 qq = qp[v4];
          float a = acc[qi];
          a = fmaf(kf[4 * v4 + 0], qq.x, a);
          a = fmaf(kf[4 * v4 + 1], qq.y, a);
          a = fmaf(kf[4 * v4 + 2], qq.z, a);
          a = fmaf(kf[4 * v4 + 3], qq.w, a);
          acc[qi] = a;
        }
      }
    }
  }
}

}  // namespace arbor

// ---- mbarrier + bulk-copy (TMA) helpers (sm_90+ PTX, used on sm_100a) -------------------
namespace arbor {

__device__ __forceinline__ uint32_t smem_u32(const void *p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t *bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(smem_u32(bar)), "r"(count));
}
__device__ __forceinline__ void mbar_fence_init() {
  asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
}
__device__ __forceinline__ void mbar_arrive_expect_tx(uint64_t *bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(smem_u32(bar)),
               "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t *bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];\n" ::"r"(smem_u32(bar)) : "memory");
}
#ifdef ARBOR_MBAR_WATCHDOG
#define mbar_wait(bar, parity) mbar_wait_impl((bar), (parity), __LINE__)
__device__ __forceinline__ void mbar_wait_impl(uint64_t *bar, uint32_t parity, int line) {
#else
__device__ __forceinline__ void mbar_wait(uint64_t *bar, uint32_t parity) {
#endif
#ifdef ARBOR_MBAR_WATCHDOG
  // debug builds (ARBOR_NVCC_FLAGS=-DARBOR_MBAR_WATCHDOG): a wait still pending after 5 s
  // prints its call site and barrier (lane 0 of the warp) and keeps waiting, so every stuck
  // role reports; after 15 s it traps — a deadlock surfaces as a CUDA error, not a hang
  unsigned long long t0;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
  bool reported = false;
  for (;;) {
    uint32_t ok;
    asm volatile(
        "{\n"
        ".reg .pred p;\n"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n"
        "selp.u32 %0, 1, 0, p;\n"
        "}\n" : "=r"(ok) : "r"(smem_u32(bar)), "r"(parity) : "memory");
    if (ok) return;
    unsigned long long t1;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t1));
    if (!reported && t1 - t0 > 5000000000ull) {
      if ((threadIdx.x & 31) == 0)
        printf("mbarrier watchdog: line %d block %d thread %d bar smem 0x%x parity %u\n", line,
               blockIdx.x, threadIdx.x, smem_u32(bar), parity);
      reported = true;
    }
    if (t1 - t0 > 15000000000ull) __trap();
  }
#endif
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "WAIT_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      "@!p bra WAIT_%=;\n"
      "}\n" ::"r"(smem_u32(bar)), "r"(parity) : "memory");
}
// Blocking wait for a role that may wait long (e.g. a consumer starved by its producer): the
// try_wait suspends the warp for up to `hint_ns` instead of returning at once, so the waiting
// warp does not spin issue slots away from the warps it waits for.
__device__ __forceinline__ void mbar_wait_sleep(uint64_t *bar, uint32_t parity, uint32_t hint_ns) {
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "WAITS_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1, %2;\n"
      "@!p bra WAITS_%=;\n"
      "}\n" ::"r"(smem_u32(bar)), "r"(parity), "r"(hint_ns) : "memory");
}
// 1-D bulk copy global → shared (TMA engine), completing `bytes` on the mbarrier.
__device__ __forceinline__ void bulk_g2s(void *dst, const void *src, uint32_t bytes, uint64_t *bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\n"
      ::"r"(smem_u32(dst)), "l"(src), "r"(bytes), "r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void named_bar_sync(int id, int threads) {
  asm volatile("bar.sync %0, %1;\n" ::"r"(id), "r"(threads) : "memory");
}

}  // namespace arbor
