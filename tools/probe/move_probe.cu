// move_probe.cu — microbenchmark for the compaction move (a6): M random (src row, dst row)
// pairs of 256-byte K and V rows (+ 2-byte pos tags) in 1.3 GB pools, moved by
//   reg:  warps streaming 16-byte pieces through registers (evict.cu move_rows, U rows/lane group)
//   bulk: TMA bulk copies global → shared → global (cp.async.bulk, one lane per row, per-lane
//         ring of S slots, per-slot mbarrier for the load, bulk async-groups for the store)
// Prints GB/s of algorithmic traffic (4 × 256 B + 4 B per pair).  Build + run:
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/move_probe tools/probe/move_probe.cu && /tmp/move_probe
#include <cstdio>
#include <cstdint>
#include <cstdlib>
#include <vector>
#include <algorithm>
#include <random>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e_ = (x); if (e_ != cudaSuccess) { printf("%s:%d %s\n", __FILE__, __LINE__, cudaGetErrorString(e_)); exit(1); } } while (0)

constexpr int RB = 256;

template <int U>
__global__ void __launch_bounds__(512, 2) reg_move(const int2 *__restrict__ jobs, int M, char *kp, char *vp,
                                                   int16_t *pos, int *ctr) {
  const int lane = threadIdx.x & 31;
  const int piece = lane & 15, sub = lane >> 4;
  const int gw = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int nw = (gridDim.x * blockDim.x) >> 5;
  // chunks of 64 jobs per warp, strided
  for (int c0 = gw * 64; c0 < M; c0 += nw * 64) {
    const int end = min(c0 + 64, M);
    for (int i0 = c0; i0 < end; i0 += 2 * U) {
      uint4 bk[U], bv[U];
      int sr[U], dr[U];
      int16_t pt[U];
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const int i = i0 + 2 * u + sub;
        sr[u] = -1;
        if (i < end) { const int2 j = jobs[i]; sr[u] = j.x; dr[u] = j.y; }
        if (sr[u] >= 0) {
          const int64_t off = static_cast<int64_t>(sr[u]) * RB + piece * 16;
          bk[u] = *reinterpret_cast<const uint4 *>(kp + off);
          bv[u] = *reinterpret_cast<const uint4 *>(vp + off);
          if (piece == 0) pt[u] = pos[sr[u]];
        }
      }
#pragma unroll
      for (int u = 0; u < U; ++u) {
        if (sr[u] >= 0) {
          const int64_t off = static_cast<int64_t>(dr[u]) * RB + piece * 16;
          *reinterpret_cast<uint4 *>(kp + off) = bk[u];
          *reinterpret_cast<uint4 *>(vp + off) = bv[u];
          if (piece == 0) pos[dr[u]] = pt[u];
        }
      }
    }
  }
}

__device__ __forceinline__ uint32_t su32(const void *p) { return static_cast<uint32_t>(__cvta_generic_to_shared(p)); }

// S slots per lane, stores lag the loads by L = S/2 rounds; W mover warps per CTA; each lane
// moves its own rows through its ring (bulk async-groups are per thread)
template <int S>
__global__ void bulk_move(const int2 *__restrict__ jobs, int M, char *kp, char *vp, int16_t *pos, int W) {
  constexpr int L = S / 2;
  extern __shared__ __align__(128) unsigned char sm[];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  unsigned char *ring = sm + static_cast<size_t>(warp) * 32 * S * 2 * RB;   // [S][32 lanes][K|V][256]
  uint64_t *bars = reinterpret_cast<uint64_t *>(sm + static_cast<size_t>(W) * 32 * S * 2 * RB) + (warp * 32 + lane) * S;
  for (int s = 0; s < S; ++s) asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(&bars[s])));
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  __syncwarp();
  const int gw = blockIdx.x * W + warp, nw = gridDim.x * W;
  int16_t ptag[S];
  int dst[S];
  const int rounds = (M + 32 * nw - 1) / (32 * nw);
  for (int r0 = 0; r0 < rounds + L; r0 += S) {
#pragma unroll
    for (int s = 0; s < S; ++s) {
      const int r = r0 + s;
      if (r < rounds) {
        const int i = (gw + r * nw) * 32 + lane;
        // slot s was last used by round r − S, stored at iteration r − S + L: S − L − 1 groups since
        asm volatile("cp.async.bulk.wait_group.read %0;" ::"n"(S - L - 1) : "memory");
        dst[s] = -1;
        if (i < M) {
          const int2 j = jobs[i];
          unsigned char *sk = ring + (static_cast<size_t>(s) * 32 + lane) * 2 * RB;
          const uint32_t b = su32(&bars[s]);
          asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(b), "r"(2 * RB) : "memory");
          asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                       ::"r"(su32(sk)), "l"(kp + static_cast<int64_t>(j.x) * RB), "n"(RB), "r"(b) : "memory");
          asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                       ::"r"(su32(sk + RB)), "l"(vp + static_cast<int64_t>(j.x) * RB), "n"(RB), "r"(b) : "memory");
          ptag[s] = pos[j.x];
          dst[s] = j.y;
        }
      }
      const int q = r - L;
      const int qs = (s - L + S) % S;
      if (q >= 0 && q < rounds) {
        if (dst[qs] >= 0) {
          const uint32_t b = su32(&bars[qs]);
          const uint32_t par = (q / S) & 1;
          asm volatile("{\n.reg .pred p;\nW_%=:\nmbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n@!p bra W_%=;\n}\n"
                       ::"r"(b), "r"(par) : "memory");
          unsigned char *sk = ring + (static_cast<size_t>(qs) * 32 + lane) * 2 * RB;
          asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;"
                       ::"l"(kp + static_cast<int64_t>(dst[qs]) * RB), "r"(su32(sk)), "n"(RB) : "memory");
          asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;"
                       ::"l"(vp + static_cast<int64_t>(dst[qs]) * RB), "r"(su32(sk + RB)), "n"(RB) : "memory");
          pos[dst[qs]] = ptag[qs];
        }
      }
      asm volatile("cp.async.bulk.commit_group;" ::: "memory");
    }
  }
  asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
}

int main(int argc, char **argv) {
  const int64_t rows = (1300ll << 20) / RB;
  const int M = argc > 1 ? atoi(argv[1]) : 560000;
  char *kp, *vp;
  int16_t *pos;
  int2 *jobs;
  int *ctr;
  CK(cudaMalloc(&kp, rows * RB));
  CK(cudaMalloc(&vp, rows * RB));
  CK(cudaMalloc(&pos, rows * 2));
  CK(cudaMalloc(&jobs, M * sizeof(int2)));
  CK(cudaMalloc(&ctr, 4));
  char *flush;
  CK(cudaMalloc(&flush, 512 << 20));
  std::mt19937_64 g(1);
  std::vector<int> perm(rows);
  for (int64_t i = 0; i < rows; ++i) perm[i] = static_cast<int>(i);
  for (int i = 0; i < 2 * M; ++i) std::swap(perm[i], perm[i + g() % (rows - i)]);
  std::vector<int2> hj(M);
  const int mode = argc > 2 ? atoi(argv[2]) : 0;
  if (mode == 2) {
    // C2-like: node-rows of 128 slots in 8 random 16-row page-heads; 14 moves per node-row
    // from slots [0, 96) into the window [96, 128), node-row after node-row
    const int64_t heads = rows / 16;
    std::vector<int> hp(heads);
    for (int64_t i = 0; i < heads; ++i) hp[i] = static_cast<int>(i);
    const int nr = (M + 13) / 14;
    for (int i = 0; i < 8 * nr; ++i) std::swap(hp[i], hp[i + g() % (heads - i)]);
    int m = 0;
    for (int r = 0; r < nr && m < M; ++r) {
      int sl[128];
      for (int i = 0; i < 128; ++i) sl[i] = i;
      for (int i = 0; i < 14; ++i) std::swap(sl[i], sl[i + g() % (96 - i)]);
      for (int i = 0; i < 14; ++i) std::swap(sl[96 + i], sl[96 + i + g() % (32 - i)]);
      std::sort(sl, sl + 14);
      std::sort(sl + 96, sl + 110);
      for (int i = 0; i < 14 && m < M; ++i, ++m) {
        const int a = sl[i], b = sl[96 + i];
        hj[m] = make_int2(hp[8 * r + a / 16] * 16 + a % 16, hp[8 * r + b / 16] * 16 + b % 16);
      }
    }
  } else {
    for (int i = 0; i < M; ++i) hj[i] = make_int2(perm[i], perm[M + i]);
    // page-local variant: sort jobs by src (rows of one page-head together)
    if (mode == 1) std::sort(hj.begin(), hj.end(), [](int2 a, int2 b) { return a.x < b.x; });
  }
  CK(cudaMemcpy(jobs, hj.data(), M * sizeof(int2), cudaMemcpyHostToDevice));
  int sms;
  CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0));
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  const double bytes = static_cast<double>(M) * (4 * RB + 4);
  auto timeit = [&](const char *name, auto launch) {
    float best = 1e9, sum = 0;
    for (int it = 0; it < 12; ++it) {
      CK(cudaMemsetAsync(flush, it, 512 << 20));
      cudaEventRecord(e0);
      launch();
      cudaEventRecord(e1);
      CK(cudaEventSynchronize(e1));
      float ms;
      cudaEventElapsedTime(&ms, e0, e1);
      if (it >= 2) { best = std::min(best, ms); sum += ms; }
    }
    CK(cudaGetLastError());
    printf("%-28s best %8.2f us  mean %8.2f us  %7.1f GB/s (best)\n", name, best * 1e3, sum / 10 * 1e3,
           bytes / (best * 1e-3) / 1e9);
  };
  for (int wps : {32, 16, 12, 8, 6}) {   // moving warps per SM (2 CTAs)
    char nm[64];
    snprintf(nm, sizeof nm, "reg U=4 %d warps/SM", wps);
    timeit(nm, [&] { reg_move<4><<<sms * 2, wps * 16>>>(jobs, M, kp, vp, pos, ctr); });
    snprintf(nm, sizeof nm, "reg U=6 %d warps/SM", wps);
    timeit(nm, [&] { reg_move<6><<<sms * 2, wps * 16>>>(jobs, M, kp, vp, pos, ctr); });
  }
  if (argc > 3) return 0;
  for (int W : {2, 3, 4}) {
    for (int S : {3, 4}) {
      const size_t smem = static_cast<size_t>(W) * 32 * S * 2 * RB + W * 32 * S * 8;
      if (smem > 227 * 1024) continue;
      char nm[64];
      auto kfn = S == 4 ? bulk_move<4> : bulk_move<3>;
      CK(cudaFuncSetAttribute(kfn, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem)));
      for (int cps : {1, 2}) {
        if (smem * cps > 227 * 1024) continue;
        snprintf(nm, sizeof nm, "bulk W=%d S=%d ctas/sm=%d (%zuKB)", W, S, cps, smem >> 10);
        timeit(nm, [&] { kfn<<<sms * cps, W * 32, smem>>>(jobs, M, kp, vp, pos, W); });
      }
    }
  }
  return 0;
}
