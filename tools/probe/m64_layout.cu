// Probe: where does tcgen05.mma (cta_group::1, kind::f16, M = 64, N = 128) put the rows of D
// in TMEM?  A[m][0] = m + 1, A[m][k>0] = 0; B[n][0] = 1, B[n][k>0] = 0  =>  D[m][n] = m + 1.
// Dumps all 128 lanes x 128 columns.   nvcc -gencode arch=compute_100a,code=sm_100a m64_layout.cu
#include <cstdio>
#include <cstdint>
#include <cuda_bf16.h>

__device__ __forceinline__ uint32_t smem_u32(const void *p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ uint64_t sw128_desc(uint32_t saddr, uint32_t lbo, uint32_t sbo) {
  return static_cast<uint64_t>((saddr >> 4) & 0x3FFFu) |
         (static_cast<uint64_t>((lbo >> 4) & 0x3FFFu) << 16) |
         (static_cast<uint64_t>((sbo >> 4) & 0x3FFFu) << 32) | (1ull << 46) | (2ull << 61);
}
__host__ __device__ constexpr uint32_t bf16_idesc(int M, int N, int a_mn, int b_mn) {
  return (1u << 4) | (1u << 7) | (1u << 10) | (static_cast<uint32_t>(a_mn) << 15) |
         (static_cast<uint32_t>(b_mn) << 16) | (static_cast<uint32_t>(N >> 3) << 17) |
         (static_cast<uint32_t>(M >> 4) << 24);
}
// element (row r, col c) of a [rows][64] bf16 K-major SW128 tile (128-B rows, 8-row atoms)
__device__ __forceinline__ int sw_off(int r, int c) {
  const int chunk = (c >> 3) ^ (r & 7);
  return r * 128 + chunk * 16 + (c & 7) * 2;
}

__global__ void probe(float *out, int variant) {
  extern __shared__ __align__(1024) unsigned char sm[];
  unsigned char *A = sm;            // [64 rows][64 k]   8 KB
  unsigned char *B = sm + 8192;     // [128 rows][64 k]  16 KB   (K-major)
  unsigned char *V = sm + 8192 + 16384;   // variant 1: B as MN-major [2 d-halves][64 keys][64 d]
  __shared__ __align__(8) uint64_t bar;
  __shared__ uint32_t tbase;
  const int tid = threadIdx.x, warp = tid >> 5;
  for (int i = tid; i < (8192 + 16384 + 16384) / 2; i += blockDim.x)
    reinterpret_cast<__nv_bfloat16 *>(sm)[i] = __float2bfloat16(0.f);
  __syncthreads();
  if (tid < 64) *reinterpret_cast<__nv_bfloat16 *>(A + sw_off(tid, 0)) = __float2bfloat16(float(tid + 1));
  if (variant == 0) {
    if (tid < 128) *reinterpret_cast<__nv_bfloat16 *>(B + sw_off(tid, 0)) = __float2bfloat16(1.f);
  } else {
    // V[key][d] with key = k index, d = n index: MN-major B (N contiguous). Set V[0][d] = d + 1
    // (d-half h = d / 64 at offset h*8192: [64 keys][64 d] SW128 per half) => D[m][n] = (m+1)(n+1)
    if (tid < 128) {
      const int h = tid >> 6, d = tid & 63;
      *reinterpret_cast<__nv_bfloat16 *>(V + h * 8192 + sw_off(0, d)) = __float2bfloat16(float(tid + 1));
    }
  }
  asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
  if (tid == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;\n" ::"r"(smem_u32(&bar)));
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 128;\n" ::"r"(smem_u32(&tbase)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;\n");
  }
  asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
  const uint32_t tmem = tbase;
  if (tid == 0) {
    const uint32_t idesc = bf16_idesc(64, 128, 0, variant);
    for (int kk = 0; kk < 4; ++kk) {
      const uint64_t ad = sw128_desc(smem_u32(A) + kk * 32, 16, 1024);
      uint64_t bd;
      if (variant == 0) bd = sw128_desc(smem_u32(B) + kk * 32, 16, 1024);
      else bd = sw128_desc(smem_u32(V) + kk * 2048, 8192, 1024);   // 16 keys x 128 B per step
      asm volatile("{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\n"
                   "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n}\n" ::"r"(tmem),
                   "l"(ad), "l"(bd), "r"(idesc), "r"(kk));
    }
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n"
                 ::"r"(smem_u32(&bar)) : "memory");
  }
  // wait
  asm volatile("{\n.reg .pred p;\nW: mbarrier.try_wait.parity.shared::cta.b64 p, [%0], 0;\n@!p bra W;\n}\n"
               ::"r"(smem_u32(&bar)) : "memory");
  asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
  for (int c = 0; c < 128; c += 8) {
    uint32_t r[8];
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];\n"
                 : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7])
                 : "r"(tmem + (static_cast<uint32_t>(warp * 32) << 16) + c));
    asm volatile("tcgen05.wait::ld.sync.aligned;\n" ::: "memory");
    for (int i = 0; i < 8; ++i) out[tid * 128 + c + i] = __uint_as_float(r[i]);
  }
  asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory");
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 128;\n" ::"r"(tmem));
}

int main() {
  float *d, h[128 * 128];
  cudaMalloc(&d, sizeof(h));
  for (int variant = 0; variant < 2; ++variant) {
    cudaMemset(d, 0, sizeof(h));
    cudaFuncSetAttribute(probe, cudaFuncAttributeMaxDynamicSharedMemorySize, 48 * 1024);
    probe<<<1, 128, 48 * 1024>>>(d, variant);
    cudaError_t e = cudaDeviceSynchronize();
    cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
    printf("variant %d (%s): %s\n", variant, variant ? "B MN-major: D = (m+1)(n+1)" : "B K-major: D = m+1",
           cudaGetErrorString(e));
    for (int lane = 0; lane < 128; ++lane) {
      printf("lane %3d:", lane);
      for (int c : {0, 1, 2, 63, 64, 127}) printf(" %7.0f", h[lane * 128 + c]);
      printf("\n");
    }
  }
  return 0;
}
