// attn_tc.cu — §8(a) a9 on the 5th-generation tensor cores (tcgen05 + TMEM + TMA), bf16, d = 128.
//
// Same operation as attn.cu (Q24): for every active leaf b, layer l
// and query head g (KV head h = g / G), o = Σ_t softmax_t(q·k_t/√d) v_t over the retained slots
// of Path(ℓ_b), emitted as split-softmax partials per (chunk of kAttnChunk = 64 slots, leaf) and
// merged root→leaf by attn_merge_kernel (attn.cu), plus the log2-domain logits z the fused score
// pass (score.cu) turns into A.
//
// Why tensor cores: a work tile holds up to two 64-slot chunks of one node (128 K/V rows of one
// (layer, KV head)) and the nq = (leaves sharing the node) × G query rows that read them.  Both
// products are dense contractions — S = K·Qᵀ (128 × nq × d) and Oᵀ = Vᵀ·P (d × 2nq × 128) — so
// they are issued as two tcgen05.mma chains (M = 128, N = NQ resp. 2·NQ, K = 16 per instruction)
// with fp32 accumulators in TMEM, and the CUDA cores only run the softmax.  That removes the
// issue-bound FMA/convert work of the CUDA-core kernel, which kept it far below HBM speed.
//
// CTA layout (persistent, one CTA per SM, tiles strided over CTAs):
//   warp 0      TMA producer: per page-head, two cp.async.bulk.tensor boxes (64 cols × P rows,
//               SWIZZLE_128B) for K and for V into NSK- and NSV-stage rings; q rows staged with 16-byte
//               loads into the same 128B-swizzled K-major layout; mbarrier transaction counts.
//   warp 1      TMEM allocator + MMA issuer (one thread): MMA1(k+1) is issued before MMA2(k)
//               waits for the softmax of tile k, so the S of the next tile is ready in TMEM.
//   warps 2..5  softmax + epilogue, one thread per TMEM lane (= tile row = slot, then = d index):
//               tcgen05.ld S → mask → column max / sum over each 64-slot half (shuffles + smem) →
//               z to zbuf, P (bf16) into the K-major B operand of MMA2 → tcgen05.ld Oᵀ → partials.
// Operand layouts (canonical UMMA, SWIZZLE_128B, atoms of 8 rows × 128 B, 1024-B aligned):
//   K tile  [2 d-halves][128 rows][64]   A of MMA1, K-major,  SBO 1024
//   Q tile  [2 d-halves][NQ rows][64]    B of MMA1, K-major,  SBO 1024
//   V tile  [2 d-halves][128 rows][64]   A of MMA2 = Vᵀ, MN-major, LBO 16 KB (d-halves), SBO 1024
//   P tile  [2 slot-halves][NQ][64]      B of MMA2 = Pᵀ, K-major: one softmax over all 128 slots
//                                        of the tile (both chunks), so MMA2 is 128 × NQ × 128 and
//                                        the tile leaves ONE partial (o, m, l) per query, stored
//                                        at its first chunk's pair (the plan's merge lists hold
//                                        the even chunks only, build_plan(tile_pairs)).
// Numerics: K, V, q are bf16 (exact products, fp32 accumulation); P is rounded to bf16 for the
// PV product (relative error ≤ 2^-9 per weight, inside the bf16 tolerance 2e-2); m and l are the
// fp32 column max and the fp32 sum of the unrounded exp2 values.
#include <cuda.h>

#include <cfloat>

#include "tile.cuh"

namespace arbor {
namespace {

// softmax warpgroups, each with its own TMEM S/Oᵀ buffer and P tile, taking tiles k ≡ group
// (mod kGroups).  Two by default: three (ARBOR_TC_GROUPS=3, 576 threads) measured the same
// tile rate on C3 (137.7 vs 137.0 µs closed tree, 184 vs 180 µs DPTS) — each group's softmax
// slowed from 2.3 to 3.3 µs per tile, so the SM, not the per-group chain, sets the rate
#ifndef ARBOR_TC_GROUPS
#define ARBOR_TC_GROUPS 2
#endif
constexpr int kGroups = ARBOR_TC_GROUPS;
// warps: 0 K producer, 1 MMA, 2..5 softmax group 0, 6..9 epilogue, 10.. further softmax
// groups, last: the V producer (a second TMA-issuing warp: one warp issuing every K, Q and V
// box of a tile was the C3 tile-rate limit, ~0.6-0.8 µs of issue per tile half)
constexpr int kVWarp = 6 + 4 * kGroups;
constexpr int kTcThreads = 32 * (kVWarp + 1);
constexpr int kHdrRing = 8;                           // epilogue header / column-reduction rings
constexpr int kTileRows = 128;
constexpr int kHalf = 64;                       // = kAttnChunk
constexpr uint32_t kKVBytes = kTileRows * 256;  // one K (or V) tile: 128 rows × 128 bf16
constexpr float kLog2e = 1.4426950408889634f;
constexpr int kMaxTilePages = 2 * 64 / 16;      // page size ≥ 16 on this path

static_assert(kAttnChunk == kHalf, "a tensor-core tile is two score/attention chunks");

struct TcArgs {
  PlanView pv;
  PoolView g;
  const int32_t *ptab, *kcur, *soff;
  const __nv_bfloat16 *q;
  float *partials, *zbuf;
  __nv_bfloat16 *out;              // merged output [nA][Lc][Hq][128] and LSE [nA][Lc][Hq]
  float *lse;
  unsigned int *row_done;          // [Lc·H] tiles finished per row (zero at rest)
  int layer_begin, Lc, Hq, G, T;   // T: tiles
  float scale_log2;
  long long *trace;                // debug: clock64 per (CTA, tile, event) or NULL
  int qw;                          // query rows per leaf slot in the Q tile (8, or G: dense)
};

// debug timeline (ARBOR_TC_TRACE=1): trace[(cta·64 + tile)·16 + event] = clock64 − CTA start
// compiled only into diagnostic builds (-DARBOR_TC_TRACE_BUILD)
#ifdef ARBOR_TC_TRACE_BUILD
constexpr bool kTcTrace = true;
#else
constexpr bool kTcTrace = false;
#endif
#define TC_TRACE(k, e)                                                                      \
  do {                                                                                      \
    if (kTcTrace && a.trace && (k) < 64)                                                    \
      a.trace[(static_cast<int64_t>(blockIdx.x) * 64 + (k)) * 16 + (e)] = clock64() - t_start; \
  } while (0)

// cnt: leaves (8-column query slots) of the tile; meta: bit 0 a B half exists, bit 1 the B
// half is packed (another node's chunk with its own columns [8·cntA, 8·cnt)), bits 4+: cntA;
// ntA / ntB: the half's valid slots [lo, hi) as chunk_span packs them (common.cuh)
struct TcHdr {
  int ntA, ntB, li, h, pbA, pbB, cnt, meta;
};

// ---------------------------------------------------------------- PTX wrappers
__device__ __forceinline__ void mbar_expect_tx(uint64_t *bar, uint32_t bytes) {
  asm volatile("mbarrier.expect_tx.relaxed.cta.shared::cta.b64 [%0], %1;\n" ::"r"(smem_u32(bar)),
               "r"(bytes) : "memory");
}
__device__ __forceinline__ void tma_load_2d(void *dst, const CUtensorMap *map, int x, int y,
                                            uint64_t *bar) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%2, %3}], [%4];\n" ::"r"(smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(x), "r"(y), "r"(smem_u32(bar))
      : "memory");
}
// non-blocking probe of an mbarrier phase
__device__ __forceinline__ bool mbar_test(uint64_t *bar, uint32_t parity) {
  uint32_t ok;
  asm volatile(
      "{\n.reg .pred p;\nmbarrier.test_wait.parity.shared::cta.b64 p, [%1], %2;\n"
      "selp.u32 %0, 1, 0, p;\n}\n"
      : "=r"(ok) : "r"(smem_u32(bar)), "r"(parity) : "memory");
  return ok != 0;
}
__device__ __forceinline__ void tma_load_5d(void *dst, const CUtensorMap *map, int c0, int c1,
                                            int c2, int c3, int c4, uint64_t *bar) {
  asm volatile(
      "cp.async.bulk.tensor.5d.shared::cluster.global.tile.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%2, %3, %4, %5, %6}], [%7];\n" ::"r"(smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1), "r"(c2), "r"(c3), "r"(c4),
      "r"(smem_u32(bar))
      : "memory");
}
__device__ __forceinline__ void fence_proxy_async() {
  asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
}
__device__ __forceinline__ void tc_fence_after() {
  asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
}
__device__ __forceinline__ void tc_fence_before() {
  asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory");
}
__device__ __forceinline__ void tc_commit(uint64_t *bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n"
               ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void tc_mma(uint32_t d_tmem, uint64_t adesc, uint64_t bdesc,
                                       uint32_t idesc, uint32_t accumulate) {
  asm volatile(
      "{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\n"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n}\n" ::"r"(d_tmem),
      "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accumulate));
}
// 16 consecutive fp32 columns of this thread's TMEM lane
__device__ __forceinline__ void tmem_ld16(uint32_t taddr, float (&v)[16]) {
  uint32_t r[16];
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,"
      "%15}, [%16];\n"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]),
        "=r"(r[7]), "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]),
        "=r"(r[14]), "=r"(r[15])
      : "r"(taddr));
  asm volatile("tcgen05.wait::ld.sync.aligned;\n" ::: "memory");
#pragma unroll
  for (int i = 0; i < 16; ++i) v[i] = __uint_as_float(r[i]);
}

// Shared-memory matrix descriptor, SWIZZLE_128B (sm_100 UMMA format: start>>4 [0,14),
// LBO>>4 [16,30), SBO>>4 [32,46), version 1 at bit 46, layout type 2 at [61,64)).
__device__ __forceinline__ uint64_t sw128_desc(uint32_t saddr, uint32_t lbo, uint32_t sbo) {
  return static_cast<uint64_t>((saddr >> 4) & 0x3FFFu) |
         (static_cast<uint64_t>((lbo >> 4) & 0x3FFFu) << 16) |
         (static_cast<uint64_t>((sbo >> 4) & 0x3FFFu) << 32) | (1ull << 46) | (2ull << 61);
}
// Instruction descriptor, kind::f16: D f32, A/B bf16, majors, N>>3 at [17,23), M>>4 at [24,29).
__host__ __device__ constexpr uint32_t bf16_idesc(int M, int N, int a_mn, int b_mn) {
  return (1u << 4) | (1u << 7) | (1u << 10) | (static_cast<uint32_t>(a_mn) << 15) |
         (static_cast<uint32_t>(b_mn) << 16) | (static_cast<uint32_t>(N >> 3) << 17) |
         (static_cast<uint32_t>(M >> 4) << 24);
}

__device__ __forceinline__ float fast_exp2(float x) {   // ex2.approx.ftz: 2 ulp, −inf → +0
  float y;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}

// N consecutive fp32 TMEM columns of this thread's lane (N a multiple of 8)
template <int N>
__device__ __forceinline__ void tmem_ld(uint32_t taddr, float *v) {
#pragma unroll
  for (int c = 0; c + 16 <= N; c += 16) {
    float t[16];
    tmem_ld16(taddr + c, t);
#pragma unroll
    for (int i = 0; i < 16; ++i) v[c + i] = t[i];
  }
  if constexpr (N % 16 == 8) {
    uint32_t r[8];
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];\n"
        : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7])
        : "r"(taddr + (N - 8)));
    asm volatile("tcgen05.wait::ld.sync.aligned;\n" ::: "memory");
#pragma unroll
    for (int i = 0; i < 8; ++i) v[N - 8 + i] = __uint_as_float(r[i]);
  }
}

// W (16 or 8) consecutive fp32 TMEM columns of this thread's lane
template <int W>
__device__ __forceinline__ void tmem_ldW(uint32_t taddr, float (&v)[W]) {
  if constexpr (W == 16) {
    tmem_ld16(taddr, v);
  } else {
    static_assert(W == 8, "group width");
    uint32_t r[8];
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];\n"
        : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7])
        : "r"(taddr));
    asm volatile("tcgen05.wait::ld.sync.aligned;\n" ::: "memory");
#pragma unroll
    for (int i = 0; i < 8; ++i) v[i] = __uint_as_float(r[i]);
  }
}

// Transpose-reduce of 8 columns held by every lane: afterwards each lane holds the reduction
// over all 32 lanes of column col8(lane) (9 shuffles instead of 40).
__device__ __forceinline__ int col8(int lane) {
  return ((lane >> 4) & 1) * 4 + ((lane >> 3) & 1) * 2 + ((lane >> 2) & 1);
}
template <bool kMax>
__device__ __forceinline__ float warp_reduce8(const float *v, int lane) {
  float b[4], c[2], d;
  const bool u16 = lane & 16, u8 = lane & 8, u4 = lane & 4;
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const float send = u16 ? v[i] : v[i + 4];
    const float keep = u16 ? v[i + 4] : v[i];
    const float r = __shfl_xor_sync(0xffffffffu, send, 16);
    b[i] = kMax ? fmaxf(keep, r) : keep + r;
  }
#pragma unroll
  for (int i = 0; i < 2; ++i) {
    const float send = u8 ? b[i] : b[i + 2];
    const float keep = u8 ? b[i + 2] : b[i];
    const float r = __shfl_xor_sync(0xffffffffu, send, 8);
    c[i] = kMax ? fmaxf(keep, r) : keep + r;
  }
  {
    const float send = u4 ? c[0] : c[1];
    const float keep = u4 ? c[1] : c[0];
    const float r = __shfl_xor_sync(0xffffffffu, send, 4);
    d = kMax ? fmaxf(keep, r) : keep + r;
  }
#pragma unroll
  for (int o = 2; o; o >>= 1) {
    const float r = __shfl_xor_sync(0xffffffffu, d, o);
    d = kMax ? fmaxf(d, r) : d + r;
  }
  return d;
}

// Transpose-reduce of 16 columns held by every lane of a warp: after the butterfly each lane
// holds the reduction over all 32 lanes of column col16(lane) (16 shuffles instead of 80).
__device__ __forceinline__ int col16(int lane) {
  return ((lane >> 4) & 1) * 8 + ((lane >> 3) & 1) * 4 + ((lane >> 2) & 1) * 2 + ((lane >> 1) & 1);
}
template <bool kMax>
__device__ __forceinline__ float warp_reduce16(const float *v, int lane) {
  float a[8], b[4], c[2], d;
  const bool u16 = lane & 16, u8 = lane & 8, u4 = lane & 4, u2 = lane & 2;
#pragma unroll
  for (int i = 0; i < 8; ++i) {
    const float send = u16 ? v[i] : v[i + 8];
    const float keep = u16 ? v[i + 8] : v[i];
    const float r = __shfl_xor_sync(0xffffffffu, send, 16);
    a[i] = kMax ? fmaxf(keep, r) : keep + r;
  }
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const float send = u8 ? a[i] : a[i + 4];
    const float keep = u8 ? a[i + 4] : a[i];
    const float r = __shfl_xor_sync(0xffffffffu, send, 8);
    b[i] = kMax ? fmaxf(keep, r) : keep + r;
  }
#pragma unroll
  for (int i = 0; i < 2; ++i) {
    const float send = u4 ? b[i] : b[i + 2];
    const float keep = u4 ? b[i + 2] : b[i];
    const float r = __shfl_xor_sync(0xffffffffu, send, 4);
    c[i] = kMax ? fmaxf(keep, r) : keep + r;
  }
  {
    const float send = u2 ? c[0] : c[1];
    const float keep = u2 ? c[1] : c[0];
    const float r = __shfl_xor_sync(0xffffffffu, send, 2);
    d = kMax ? fmaxf(keep, r) : keep + r;
  }
  const float r = __shfl_xor_sync(0xffffffffu, d, 1);
  return kMax ? fmaxf(d, r) : d + r;
}

#ifdef ARBOR_TC_GW16
template <int NQ> constexpr int kW = NQ % 16 == 0 ? 16 : 8;   // reduction group width
#else
// reduction group width: 8 columns (two leaves of G = 4) — most tiles hold one or two leaves,
// whose columns a 16-wide group would process mostly masked
template <int NQ> constexpr int kW = 8;
#endif
template <int NQ>
__device__ __forceinline__ int colW(int lane) { return kW<NQ> == 16 ? col16(lane) : col8(lane); }
template <int W, bool kMax>
__device__ __forceinline__ float warp_reduceW(const float *v, int lane) {
  if constexpr (W == 16) return warp_reduce16<kMax>(v, lane);
  else return warp_reduce8<kMax>(v, lane);
}
// valid columns of an item with cnt leaves: a qw-row query slot per leaf (qw = 8, or G for
// dense slots), G q heads used per slot (cnt ≤ 6, qw ≤ 8: ≤ 48 bits)
__device__ __forceinline__ unsigned long long colmask(int cnt, int G, int qw) {
  const unsigned long long slot = (1ull << G) - 1ull;
  unsigned long long m = 0ull;
  for (int j = 0; j < cnt; ++j) m |= slot << (j * qw);
  return m;
}

constexpr int gcd_c(int a, int b) { return b == 0 ? a : gcd_c(b, a % b); }
constexpr int lcm_c(int a, int b) { return a / gcd_c(a, b) * b; }

// kGroups buffers of [S: NQ cols | Oᵀ: NQ cols]
template <int NQ>
constexpr int tmem_cols() {
  constexpr int c = 2 * kGroups * NQ;
  return c <= 32 ? 32 : c <= 64 ? 64 : c <= 128 ? 128 : c <= 256 ? 256 : 512;
}

// Dynamic smem: NSK K stages [K | Q], NSV V stages, kGroups P tiles (all 1024-B aligned).
template <int NQ, int NSK, int NSV>
struct TcSmem {
  static constexpr uint32_t kQ = NQ * 256;                    // Q tile bytes
  static constexpr uint32_t kKS = kKVBytes + kQ;              // one K stage: K | Q
  static constexpr uint32_t kVBase = NSK * kKS;               // first V stage
  static constexpr uint32_t kP = NQ * 256;                    // P tile bytes (NQ rows × 128 slots)
  static constexpr uint32_t kPBase = kVBase + NSV * kKVBytes;
  static constexpr uint32_t kBytes = kPBase + kGroups * kP;
  static constexpr uint32_t kAlloc = kBytes + 1024;           // + alignment slack
  // per-tile header ring: slot k is rewritten at K(k + kRing)'s issue, which needs
  // MMA1(k + kRing − NSK) complete ← MMA2(k + kRing − NSK − kGroups) issued ← softmax of that
  // tile done: kRing ≥ NSK + kGroups keeps it past softmax(k) (and the V issue of tile k)
  static constexpr int kRing = 8;
  static_assert(kRing >= NSK + kGroups && kRing >= NSV + kGroups, "header ring");
};

template <int NQ, int NSK, int NSV>
__global__ void __launch_bounds__(kTcThreads, 1)
attn_tc_kernel(const __grid_constant__ CUtensorMap tmk, const __grid_constant__ CUtensorMap tmv,
               const __grid_constant__ CUtensorMap tmk4, const __grid_constant__ CUtensorMap tmv4,
               const __grid_constant__ CUtensorMap tmq, TcArgs a) {
  using S = TcSmem<NQ, NSK, NSV>;
  constexpr int RING = S::kRing;
  extern __shared__ unsigned char sm_raw[];
  unsigned char *sm = reinterpret_cast<unsigned char *>(
      (reinterpret_cast<uintptr_t>(sm_raw) + 1023) & ~static_cast<uintptr_t>(1023));
  unsigned char *Pbuf = sm + S::kPBase;
  auto Kst = [&](int s) { return sm + s * S::kKS; };                 // K stage s (Q after K)
  auto Vst = [&](int s) { return sm + S::kVBase + s * kKVBytes; };  // V stage s
  // K (+ q rows) and V of a stage have their own barriers: K is free again once MMA1 has
  // read it, V only after MMA2, so the next K loads go out ~1.5 µs earlier
  // The full barriers the softmax groups wait on are split by (stage, group): tile k arms
  // full_k[k % NSK][k % kGroups] (and full_v likewise), whose consecutive tiles are LK
  // (LV) = lcm(stages, kGroups) apart, so each is waited by ONE group in tile order — with
  // kGroups not dividing the stage count a shared full barrier could be waited two phases
  // early (a fresh barrier reads its "previous" phase as complete: group 2's first tile,
  // k = 2 on stage 0, passed before K(0) landed — the 3-group hang).
  constexpr int LK = lcm_c(NSK, kGroups), LV = lcm_c(NSV, kGroups);
  __shared__ __align__(8) uint64_t full_k[NSK][kGroups], empty_k[NSK], full_v[NSV][kGroups],
      empty_v[NSV];
  // kcons[s][g]: the softmax of tile k (stage s, group g) has passed its full_k wait (128
  // arrivals).  K(j) is issued only after kcons of tile j − LK (the previous tile on its full
  // barrier), so a full barrier is never a phase ahead of a
  // softmax wait on it (no parity aliasing, for any NSK)
  __shared__ __align__(8) uint64_t kcons[NSK][kGroups];
  __shared__ __align__(8) uint64_t s_full[kGroups], s_empty[kGroups], p_full[kGroups],
      o_full[kGroups], o_empty[kGroups];
  // per-tile header and page list, ring of RING = 2·max(NSK, NSV) tiles (written at K issue;
  // read by the V issue, the softmax and — via ohdr — the epilogue; slot k is rewritten by
  // tile k + RING, whose K issue needs MMA1(k + RING − NSK), i.e. MMA2(k) issued, i.e.
  // softmax(k) done; K issue runs < RING tiles ahead of V issue)
  __shared__ TcHdr hdr[RING];
  // producer progress between the two TMA warps: K issued for tiles < kk_k_pub (their hdr and
  // vpage written first); V issued for tiles < kk_v_pub (the K producer's ring bound)
  __shared__ volatile int kk_k_pub, kk_v_pub;
  __shared__ int vpage[RING][kMaxTilePages];
  __shared__ TcHdr ohdr[kHdrRing];                      // tile k's header for the epilogue warps
  // column max / sum of each warp quadrant, ring of kHdrRing tiles (the epilogue warps read
  // tile k's before releasing Oᵀ buffer k % kGroups; softmax(k + 8) writes after o_full of
  // k + 8 − kGroups, which needed epilogue(k + 8 − 2·kGroups) ≥ epilogue(k))
  __shared__ float red_m[kHdrRing][4][NQ], red_l[kHdrRing][4][NQ];
  // column n of a tile = leaf slot j = n / qw, q head g = n % qw: col_j[n] = j and
  // col_js[n] = j·SP + g (SP = Lc·H·G: the pair stride of zbuf / partials in (l, h, g) units);
  // launch constants, so the per-column address math needs no division
  __shared__ int col_j[NQ], col_js[NQ];
  __shared__ uint32_t tmem_base_sh;

  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const long long t_start = clock64();
  if (kTcTrace && a.trace && threadIdx.x == 0) {
    unsigned long long g0;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(g0));
    a.trace[(static_cast<int64_t>(blockIdx.x) * 64 + 63) * 16 + 0] = static_cast<long long>(g0);
  }
  const int HL = a.g.H * a.Lc;
  const int total = a.T * HL;
  const int ntiles = total > static_cast<int>(blockIdx.x)
                         ? (total - 1 - static_cast<int>(blockIdx.x)) / gridDim.x + 1 : 0;
  const int P = a.g.P;
  const int lgP = 31 - __clz(P);

  // ---- producer state (warp 0).  Everything the producer needs per tile is loaded
  // lane-parallel for 32 tiles at a time (lane i: tile k0 + i) before any of those tiles'
  // TMA traffic is in flight (a plain global load issued behind ~200 KB of in-flight TMA data
  // per SM waits ~2 µs): the tile's self-contained record (node, chunk, pair bases, leaf
  // ids — host-built, so it is read before griddepcontrol.wait), then k_cur and the page ids
  // (written by earlier kernels, so after it).
  int b_c0 = 0, b_pbA = 0, b_pbB = -1, b_cnt = 0, b_ntA = 0, b_ntB = 0, b_node = 0;
  int b_nodeB = -1, b_c0B = 0, b_cntB = 0;
  int b_leaf[kLeavesPerItem];
  int b_page[kMaxTilePages];
  auto load_rec = [&](int k0) {
    const int kk = k0 + lane;
    if (kk < ntiles) {
      const int it = blockIdx.x + kk * gridDim.x;
      const int4 *r = a.pv.tl_rec + static_cast<int64_t>(it / HL) * (kTileRecInts / 4);
      const int4 r0 = r[0], r1 = r[1], r2 = r[2], r3 = r[3];
      b_node = r0.x; b_c0 = r0.y; b_pbA = r0.z; b_cnt = r0.w;
      b_nodeB = r1.x; b_c0B = r1.y; b_pbB = r1.z; b_cntB = r1.w;
      b_leaf[0] = r2.x; b_leaf[1] = r2.y; b_leaf[2] = r2.z; b_leaf[3] = r2.w;
      b_leaf[4] = r3.x; b_leaf[5] = r3.y;
    }
  };
  auto load_state = [&](int k0) {
    const int kk = k0 + lane;
    if (kk < ntiles) {
      const int kc = a.kcur[b_node], so = a.soff[b_node];
      const bool same = b_nodeB == b_node;
      const int kcB = b_nodeB < 0 ? 0 : (same ? kc : a.kcur[b_nodeB]);
      const int soB = b_nodeB < 0 ? 0 : (same ? so : a.soff[b_nodeB]);
      // a half's pages are loaded from its first page up to the one holding slot hi − 1;
      // the slots below lo (stale pages before soff, Q23*) are masked, not skipped
      b_ntA = chunk_span(so, kc, b_c0, kHalf);
      b_ntB = b_nodeB >= 0 ? chunk_span(soB, kcB, b_c0B, kHalf) : 0;
      const int pgA = (span_hi(b_ntA) + P - 1) >> lgP, pgB = (span_hi(b_ntB) + P - 1) >> lgP;
      const int ppH = kHalf >> lgP;   // pages per 64-slot half
      const int32_t *ptA = a.ptab + static_cast<int64_t>(b_node) * a.g.MPN + (b_c0 >> lgP);
      const int32_t *ptB = a.ptab + static_cast<int64_t>(b_nodeB < 0 ? 0 : b_nodeB) * a.g.MPN + (b_c0B >> lgP);
#pragma unroll
      for (int i = 0; i < kMaxTilePages; ++i) {
        const int half = i >= ppH, pi = i - half * ppH;
        b_page[i] = (pi < (half ? pgB : pgA)) ? (half ? ptB[pi] : ptA[pi]) : 0;
      }
    }
  };
  static_assert(kLeavesPerItem == 6, "tile record layout");
  if (warp != 0) {
    // zero V, Q and P once: MMA2 reads every V row (0·v must stay 0, so rows never loaded
    // must be finite) and the off-half rows of the Pᵀ tile are never written again
    for (int s = 0; s < NSV; ++s)
      for (uint32_t i = (tid - 32) * 16; i < kKVBytes; i += (kTcThreads - 32) * 16)
        *reinterpret_cast<uint4 *>(Vst(s) + i) = make_uint4(0, 0, 0, 0);
    for (int s = 0; s < NSK; ++s)
      for (uint32_t i = (tid - 32) * 16; i < S::kQ; i += (kTcThreads - 32) * 16)
        *reinterpret_cast<uint4 *>(Kst(s) + kKVBytes + i) = make_uint4(0, 0, 0, 0);
    for (uint32_t i = (tid - 32) * 16; i < kGroups * S::kP; i += (kTcThreads - 32) * 16)
      *reinterpret_cast<uint4 *>(Pbuf + i) = make_uint4(0, 0, 0, 0);
    fence_proxy_async();
  }
  if (tid >= 64 && tid < 64 + NQ) {
    const int n = tid - 64, j = n / a.qw;
    col_j[n] = j;
    col_js[n] = j * (a.Lc * a.g.H * a.G) + (n - j * a.qw);
  }
  if (tid == 32) {
    kk_k_pub = 0;
    kk_v_pub = 0;
    for (int s = 0; s < NSK; ++s) {
      for (int g = 0; g < kGroups; ++g) {
        mbar_init(&full_k[s][g], 1);
        mbar_init(&kcons[s][g], 128);   // the 4 warps of one softmax group
      }
      mbar_init(&empty_k[s], 1);
    }
    for (int s = 0; s < NSV; ++s) {
      for (int g = 0; g < kGroups; ++g) mbar_init(&full_v[s][g], 1);
      mbar_init(&empty_v[s], 1);
    }
    for (int b = 0; b < kGroups; ++b) {
      mbar_init(&s_full[b], 1);
      mbar_init(&p_full[b], 128);   // the 4 softmax warps
      mbar_init(&o_full[b], 1);
      mbar_init(&s_empty[b], 128);
      mbar_init(&o_empty[b], 128);  // the 4 epilogue warps
    }
    mbar_fence_init();
  }
  if (warp == 1) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;\n" ::"r"(
                     smem_u32(&tmem_base_sh)), "r"(tmem_cols<NQ>()));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;\n");
  }
  if (warp == 0) {
    if (lane == 0) {
      asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&tmk)) : "memory");
      asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&tmv)) : "memory");
      asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&tmk4)) : "memory");
      asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&tmv4)) : "memory");
      asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&tmq)) : "memory");
    }
    load_rec(0);   // host-built plan records: uploaded before this kernel was enqueued
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = tmem_base_sh;
  pdl_wait();   // everything above overlapped the previous kernel's tail
  pdl_trigger();

  if (warp == 0) {
    // ------------------------------------------------------------- TMA producer
    // Two cursors: K (+ q rows) of tile kk_k goes out as soon as K stage kk_k % NSK is free
    // (MMA1 of tile kk_k − NSK done), V of tile kk_v once V stage kk_v % NSV is (MMA2 of
    // kk_v − NSV done); K runs < RING tiles ahead of V.  Non-blocking polls, lane 0's view.
    const int ppH = kHalf >> lgP;
    int kk_k = 0, kk_v = 0;
    if (ntiles > 0) load_state(0);
#ifdef ARBOR_MBAR_WATCHDOG
    unsigned long long wd_t0 = 0;
    int wd_k = -1, wd_v = -1;
#endif
    while (kk_k < ntiles) {
      kk_v = __shfl_sync(0xffffffffu, kk_v_pub, 0);
#ifdef ARBOR_MBAR_WATCHDOG
      {
        unsigned long long t;
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
        if (kk_k != wd_k || kk_v != wd_v) { wd_k = kk_k; wd_v = kk_v; wd_t0 = t; }
        else if (wd_t0 && t - wd_t0 > 5000000000ull) {
          if (lane == 0)
            printf("producer stuck: block %d ntiles %d kk_k %d kk_v %d empty_k %d kcons %d empty_v %d\n",
                   blockIdx.x, ntiles, kk_k, kk_v,
                   (int)mbar_test(&empty_k[kk_k % NSK], ((kk_k / NSK) & 1u) ^ 1u),
                   (int)mbar_test(&kcons[kk_k % NSK][kk_k % kGroups], ((kk_k / LK) & 1u) ^ 1u),
                   (int)mbar_test(&empty_v[kk_v % NSV], ((kk_v / NSV) & 1u) ^ 1u));
          wd_t0 = 0;
        }
      }
#endif
      bool go_k = false, go_v = false;
      if (kk_k < ntiles && kk_k < kk_v + RING) {
        // K(j) may land only after softmax(j − NSK) has passed its full_k wait (kcons):
        // otherwise K(j) could complete full_k's NEXT phase of the same parity before
        // softmax(j − NSK) waits, and that wait would then block on K(j + NSK), which needs
        // MMA1(j) ← s_empty(j − 2) ← … softmax(j − NSK): a parity-aliasing deadlock (round 1
        // saw it as rare hangs of the 16-leaf C3 decode).  kcons has one phase per tile of
        // its stage, so the test is alias-free for any NSK (round 1 gated on s_empty by
        // TMEM buffer, which throttled NSK = 2 and could alias at NSK = 3).
        const int sk = kk_k % NSK;
        const uint32_t par = ((kk_k / NSK) & 1u) ^ 1u;
#ifdef ARBOR_TC_NOGATE   // diagnostics only: no kcons gate (can deadlock)
        const bool ok = mbar_test(&empty_k[sk], par);
#else
        const bool ok = mbar_test(&empty_k[sk], par) &&
                        mbar_test(&kcons[sk][kk_k % kGroups], ((kk_k / LK) & 1u) ^ 1u);
#endif
        go_k = __shfl_sync(0xffffffffu, ok ? 1 : 0, 0) != 0;
      }
      if (go_k) {
        const int k = kk_k;
        if ((k & 31) == 0 && k > 0) {
          load_rec(k);
          load_state(k);
        }
        const int src = k & 31;
        const int ntA = __shfl_sync(0xffffffffu, b_ntA, src);
        const int ntB = __shfl_sync(0xffffffffu, b_ntB, src);
        const int pbA = __shfl_sync(0xffffffffu, b_pbA, src);
        const int pbB = __shfl_sync(0xffffffffu, b_pbB, src);
        const int cntA = __shfl_sync(0xffffffffu, b_cnt, src);
        const int cntB = __shfl_sync(0xffffffffu, b_cntB, src);   // > 0: packed B half
        const int cnt = cntA + cntB;
        int page = 0, leaf = 0;       // lane i < pages: page i of the tile; lane i < cnt: leaf i
#pragma unroll
        for (int i = 0; i < kMaxTilePages; ++i) {
          const int v = __shfl_sync(0xffffffffu, b_page[i], src);
          if (lane == i) page = v;
        }
#pragma unroll
        for (int i = 0; i < kLeavesPerItem; ++i) {
          const int v = __shfl_sync(0xffffffffu, b_leaf[i], src);
          if (lane == i) leaf = v;
        }
        const int it = blockIdx.x + k * gridDim.x;
        const int li = (it / a.g.H) % a.Lc, h = it % a.g.H;
        const int pgA = (span_hi(ntA) + P - 1) >> lgP, pgB = (span_hi(ntB) + P - 1) >> lgP;
        const int s = k % NSK, r = k % RING;
        uint64_t *fkb = &full_k[s][k % kGroups];
        if (lane == 0) { TC_TRACE(k, 0); TC_TRACE(k, 1); }
        unsigned char *Ks = Kst(s);
        unsigned char *Qs = Ks + kKVBytes;
        if (lane == 0) {
          hdr[r] = TcHdr{ntA, ntB, li, h, pbA, pbB, cnt,
                         (pbB >= 0 ? 1 : 0) | (cntB > 0 ? 2 : 0) | (cntA << 4)};
          mbar_arrive_expect_tx(fkb, static_cast<uint32_t>(pgA + pgB) * P * 256u +
                                                static_cast<uint32_t>(cnt * a.qw) * 256u);
        }
        if (lane < kMaxTilePages) vpage[r][lane] = page;
        __syncwarp();
        const int l = a.layer_begin + li;
        const int half = lane >= ppH, pi = lane - half * ppH;
        const int pgh = half ? pgB : pgA;
        // a chunk whose pages are all present and consecutive (the usual case: pages are
        // popped in order) is fetched with one 64-row box per d-half through the 5-D view of
        // the pool; otherwise one 16-row box per page-head through the 2-D view
        const int first = __shfl_sync(0xffffffffu, page, half * ppH);
        const bool cons = lane >= 2 * ppH || pi >= pgh || page == first + pi;
        const unsigned bal = __ballot_sync(0xffffffffu, cons);
        const unsigned hmask = ((1u << ppH) - 1u) << (half * ppH);
        const bool big = lane < 2 * ppH && pgh == ppH && (bal & hmask) == hmask;
        if (big) {
          if (pi == 0) {
            const int lp = l * a.g.NP + page;
            const uint32_t dst = static_cast<uint32_t>(half * kHalf) * 128u;
            tma_load_5d(Ks + dst, &tmk4, 0, 0, 0, h, lp, fkb);
            tma_load_5d(Ks + 16384 + dst, &tmk4, 0, 1, 0, h, lp, fkb);
          }
        } else if (lane < 2 * ppH && pi < pgh) {
          const int row = static_cast<int>(pool_row(a.g, l, page, h, 0));
          const uint32_t dst = static_cast<uint32_t>(half * kHalf + pi * P) * 128u;
          tma_load_2d(Ks + dst, &tmk, 0, row, fkb);
          tma_load_2d(Ks + 16384 + dst, &tmk, 64, row, fkb);
        }
        if (lane < cnt) {
          // leaf `lane`: its G q rows (a qw-row box) → Q rows [qw·lane, qw·lane + qw)
          const int row = (leaf * a.Lc + li) * a.Hq + h * a.G;
          tma_load_2d(Qs + lane * a.qw * 128, &tmq, 0, row, fkb);
          tma_load_2d(Qs + NQ * 128 + lane * a.qw * 128, &tmq, 64, row, fkb);
        }
        if (lane == 0) TC_TRACE(k, 2);
        ++kk_k;
        __syncwarp();
        __threadfence_block();               // hdr / vpage of tile k before the count
        if (lane == 0) kk_k_pub = kk_k;
      }
    }
  } else if (warp == kVWarp) {
    // ------------------------------------------------------------- V producer
    const int ppH = kHalf >> lgP;
    int kk_v = 0;
    while (kk_v < ntiles) {
      const int kk_k = __shfl_sync(0xffffffffu, kk_k_pub, 0);
      __threadfence_block();                 // the count before the tile's hdr / vpage
      bool go_v = false;
      if (kk_v < kk_k) {
        const int sv = kk_v % NSV;
        go_v = __shfl_sync(0xffffffffu, mbar_test(&empty_v[sv], ((kk_v / NSV) & 1u) ^ 1u) ? 1 : 0, 0) != 0;
      }
      if (go_v) {
        const int k = kk_v;
        const int s = k % NSV, r = k % RING;
        const TcHdr hd = hdr[r];
        const int page = lane < kMaxTilePages ? vpage[r][lane] : 0;
        const int pgA = (span_hi(hd.ntA) + P - 1) >> lgP, pgB = (span_hi(hd.ntB) + P - 1) >> lgP;
        unsigned char *Vs = Vst(s);
        uint64_t *fvb = &full_v[s][k % kGroups];
        if (lane == 0) mbar_arrive_expect_tx(fvb, static_cast<uint32_t>(pgA + pgB) * P * 256u);
        __syncwarp();
        const int l = a.layer_begin + hd.li;
        const int half = lane >= ppH, pi = lane - half * ppH;
        const int pgh = half ? pgB : pgA;
        const int first = __shfl_sync(0xffffffffu, page, half * ppH);
        const bool cons = lane >= 2 * ppH || pi >= pgh || page == first + pi;
        const unsigned bal = __ballot_sync(0xffffffffu, cons);
        const unsigned hmask = ((1u << ppH) - 1u) << (half * ppH);
        const bool big = lane < 2 * ppH && pgh == ppH && (bal & hmask) == hmask;
        if (big) {
          if (pi == 0) {
            const int lp = l * a.g.NP + page;
            const uint32_t dst = static_cast<uint32_t>(half * kHalf) * 128u;
            tma_load_5d(Vs + dst, &tmv4, 0, 0, 0, hd.h, lp, fvb);
            tma_load_5d(Vs + 16384 + dst, &tmv4, 0, 1, 0, hd.h, lp, fvb);
          }
        } else if (lane < 2 * ppH && pi < pgh) {
          const int row = static_cast<int>(pool_row(a.g, l, page, hd.h, 0));
          const uint32_t dst = static_cast<uint32_t>(half * kHalf + pi * P) * 128u;
          tma_load_2d(Vs + dst, &tmv, 0, row, fvb);
          tma_load_2d(Vs + 16384 + dst, &tmv, 64, row, fvb);
        }
        ++kk_v;
        __syncwarp();
        if (lane == 0) kk_v_pub = kk_v;
      }
    }
  } else if (warp == 1) {
    // ------------------------------------------------------------- MMA issuer
    if (lane == 0) {
      constexpr uint32_t id1 = bf16_idesc(128, NQ, 0, 0);       // S = K · Qᵀ
      constexpr uint32_t id2 = bf16_idesc(128, NQ, 1, 0);       // Oᵀ = Vᵀ · Pᵀ
      // Two independent streams of work, issued as soon as each is ready (non-blocking
      // polls): MMA1(j) needs tile j's stage (full) and S buffer j % kGroups drained (s_empty
      // of j − kGroups); MMA2(j) needs P(j) (p_full) and Oᵀ buffer j % kGroups drained
      // (o_empty of j − kGroups).  MMA1 runs at most kGroups − 1 tiles ahead of MMA2.
      int js = 0, jo = 0;
#ifdef ARBOR_MBAR_WATCHDOG
      unsigned long long wd_t0 = 0;
      int wd_s = -1, wd_o = -1;
#endif
      while (jo < ntiles) {
#ifdef ARBOR_MBAR_WATCHDOG
        {
          unsigned long long t;
          asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
          if (js != wd_s || jo != wd_o) { wd_s = js; wd_o = jo; wd_t0 = t; }
          else if (wd_t0 && t - wd_t0 > 5000000000ull) {
            printf("mma stuck: block %d ntiles %d js %d jo %d full_k %d s_empty %d p_full %d o_empty %d\n",
                   blockIdx.x, ntiles, js, jo,
                   js < ntiles ? (int)mbar_test(&full_k[js % NSK][js % kGroups], (js / LK) & 1u) : -1,
                   js < kGroups ? 1 : (int)mbar_test(&s_empty[js % kGroups], ((js - kGroups) / kGroups) & 1u),
                   (int)mbar_test(&p_full[jo % kGroups], (jo / kGroups) & 1u),
                   jo < kGroups ? 1 : (int)mbar_test(&o_empty[jo % kGroups], ((jo - kGroups) / kGroups) & 1u));
            wd_t0 = 0;
          }
        }
#endif
#ifdef ARBOR_TC_MMA1_LOCKSTEP   // round-1 behaviour: MMA1 at most kGroups − 1 tiles ahead of MMA2
        if (js < ntiles && js <= jo + kGroups - 1 &&
#else
        // MMA1(j) waits only for its data and its S buffer: with the lock step (j ≤ MMA2's
        // index + 1) softmax(j) could not start before softmax(j − 1) had finished, which
        // serialised the two groups (round-1 design; the deadlock it was blamed on was the
        // full-barrier parity aliasing, fixed by the per-(stage, group) barriers)
        if (js < ntiles &&
#endif
            mbar_test(&full_k[js % NSK][js % kGroups], (js / LK) & 1u) &&
            (js < kGroups || mbar_test(&s_empty[js % kGroups], ((js - kGroups) / kGroups) & 1u))) {
          const int s = js % NSK, b = js % kGroups;
          TC_TRACE(js, 3);
          tc_fence_after();
          const uint32_t ks = smem_u32(Kst(s));
          const uint32_t qs = ks + kKVBytes;
#pragma unroll
          for (int kk = 0; kk < 8; ++kk) {
            const uint64_t ad = sw128_desc(ks + (kk >> 2) * 16384u + (kk & 3) * 32u, 16, 1024);
            const uint64_t bd = sw128_desc(qs + (kk >> 2) * (NQ * 128u) + (kk & 3) * 32u, 16, 1024);
            tc_mma(tmem + b * 2 * NQ, ad, bd, id1, kk > 0);
          }
          tc_commit(&s_full[b]);
          tc_commit(&empty_k[s]);            // K (and q) of this stage may be reloaded
          if (kTcTrace && a.trace) { mbar_wait(&s_full[b], (js / kGroups) & 1u); TC_TRACE(js, 12); }
          ++js;
        }
        if (jo < js && mbar_test(&p_full[jo % kGroups], (jo / kGroups) & 1u) &&
            (jo < kGroups || mbar_test(&o_empty[jo % kGroups], ((jo - kGroups) / kGroups) & 1u))) {
          const int s = jo % NSV, b = jo % kGroups;
          TC_TRACE(jo, 5);
          tc_fence_after();
          const uint32_t vs = smem_u32(Vst(s));
          const uint32_t ps = smem_u32(Pbuf + b * S::kP);
#pragma unroll
          for (int kk = 0; kk < 8; ++kk) {
            const uint64_t ad = sw128_desc(vs + kk * 2048u, 16384, 1024);
            const uint64_t bd = sw128_desc(ps + (kk >> 2) * (NQ * 128u) + (kk & 3) * 32u, 16, 1024);
            tc_mma(tmem + b * 2 * NQ + NQ, ad, bd, id2, kk > 0);
          }
          tc_commit(&o_full[b]);
          tc_commit(&empty_v[s]);
          if (kTcTrace && a.trace) { mbar_wait(&o_full[b], (jo / kGroups) & 1u); TC_TRACE(jo, 13); }
          ++jo;
        }
      }
    }
  } else if (warp < 6 || warp >= 10) {
    // ------------------------------------------------------- softmax (warps 2..5 and 10..13)
    // One thread per TMEM lane = tile row = slot.  Columns (queries) are independent, so a
    // tile is processed in groups of GW columns by a rolled loop — only the tile's own
    // columns (8 q rows per leaf), and a loop body that stays small for the instruction
    // cache whatever NQ is (a fully unrolled NQ = 48 body thrashed it).
    // Two warpgroups alternate over the tiles (group g takes k ≡ g mod 2, i.e. TMEM and P
    // buffer g): one tile's latency-bound softmax chain overlaps the next one's.
    // One column max / sum over the whole 128-slot tile (both chunks): the four warps of the
    // group combine their warp results through smem behind one 128-thread named barrier.
    constexpr int GW = kW<NQ>;
    const int grp = warp < 6 ? 0 : (warp - 6) / 4;   // warps 2..5 → 0, 10..13 → 1, 14..17 → 2
    static_assert(kGroups >= 2 && kGroups <= 3, "softmax groups");
    const int quad = warp & 3;                 // TMEM lane quadrant of this warp
    const int half = quad >> 1;                // slot half (chunk A or B) of this thread
    const int bar_id = 1 + grp;                // named barrier of this group (128 threads)
    const int trow = quad * 32 + lane;         // tile row (slot)
    const int tc = trow & (kHalf - 1);         // slot within the chunk
    const int G = a.G;
    const uint32_t lane_addr = static_cast<uint32_t>(quad * 32) << 16;
    const int SP = a.Lc * a.g.H * G;
    const int myc = colW<NQ>(lane);
    const uint32_t cb = static_cast<uint32_t>(tc * 2);
    for (int k = grp; k < ntiles; k += kGroups) {
      const int s = k % NSK, b = k % kGroups, ph = (k / kGroups) & 1;
      mbar_wait(&full_k[s][grp], (k / LK) & 1u);
      if (tid == 64) TC_TRACE(k, 7);
      const TcHdr hd = hdr[k % RING];
      mbar_arrive(&kcons[s][grp]);          // past the full_k wait: K(k + LK) may land
      const int cntA = hd.meta >> 4;
      const bool pack = (hd.meta & 2) != 0;
      // this half's query columns: a packed B half has its own, after A's
      const int qw = a.qw;
      const unsigned long long cm = (half && pack) ? colmask(hd.cnt - cntA, G, qw) << (qw * cntA)
                                                   : colmask(cntA, G, qw);
      const int lofs = (half && pack) ? cntA : 0;   // first leaf slot of this half's pair group
      const int nt = half ? hd.ntB : hd.ntA;
      const bool present = half == 0 || (hd.meta & 1);
      const int pb = half ? hd.pbB : hd.pbA;
      const bool valid = present && tc >= span_lo(nt) && tc < span_hi(nt);
      const int ngrp = (min(NQ, qw * hd.cnt) + GW - 1) / GW;
      mbar_wait(&s_full[b], ph);
      if (tid == 64) TC_TRACE(k, 8);
      tc_fence_after();
      // P buffer b was last read by MMA2(k − kGroups)
      if (k >= kGroups) mbar_wait(&o_full[b], ph ^ 1);
      // the header for the epilogue warps: ring slot k % 8 was last read by epilogue(k − 8)
      // before its o_empty arrival, which MMA2(k − kGroups) — complete, o_full above —
      // waited for (kHdrRing ≥ 2·kGroups); written earlier, right after the full_k wait, it
      // could overtake the epilogue once K runs ahead (tiles with another tile's header)
      if (half == 0 && lane == 0 && quad == 0) ohdr[k % kHdrRing] = hd;
      // P (bf16) goes to row n of slot-half `half` of the Pᵀ tile; rows of columns past the
      // tile's own keep stale values: they only feed output columns that are never stored
      // (Oᵀ column n depends on Pᵀ row n alone)
      unsigned char *Pt = Pbuf + b * S::kP + half * (NQ * 128);
      float *zr = a.zbuf + ((static_cast<int64_t>(pb) * a.Lc + hd.li) * a.g.H + hd.h) * G * kAttnChunk + tc;
#pragma unroll 1
      for (int gi = 0; gi < ngrp; ++gi) {
        const int c = gi * GW;
        float z[GW], p[GW];
        tmem_ldW<GW>(tmem + lane_addr + b * 2 * NQ + c, z);
#pragma unroll
        for (int i = 0; i < GW; ++i)
          z[i] = (valid && ((cm >> (c + i)) & 1ull)) ? z[i] * a.scale_log2 : -INFINITY;
        // column max and sum over the 128 slots: butterfly transpose-reduce in the warp, then
        // the group's four warps combine through smem (ring of 4 tiles)
        const float mw = warp_reduceW<GW, true>(z, lane);
        if (!(lane & 1)) red_m[k % kHdrRing][quad][c + myc] = mw;
        named_bar_sync(bar_id, 128);
#pragma unroll
        for (int i = 0; i < GW; ++i) {
          const float m = fmaxf(fmaxf(red_m[k % kHdrRing][0][c + i], red_m[k % kHdrRing][1][c + i]),
                                fmaxf(red_m[k % kHdrRing][2][c + i], red_m[k % kHdrRing][3][c + i]));
          p[i] = z[i] == -INFINITY ? 0.f : fast_exp2(z[i] - m);   // m = −inf only if all masked
        }
        const float lw = warp_reduceW<GW, false>(p, lane);
        if (!(lane & 1)) red_l[k % kHdrRing][quad][c + myc] = lw;
#pragma unroll
        for (int i = 0; i < GW; ++i) {
          const int r = c + i;
          *reinterpret_cast<__nv_bfloat16 *>(Pt + r * 128 + ((((cb >> 4) ^ (r & 7))) << 4) + (cb & 15)) =
              __float2bfloat16_rn(p[i]);
        }
        if (valid) {   // logits for the fused score pass: zbuf[pair][li][h][g][slot]
#pragma unroll
          for (int i = 0; i < GW; ++i) {
            const int n = c + i;
            if ((cm >> n) & 1ull)
              zr[static_cast<int64_t>(col_js[n] - lofs * SP) * kAttnChunk] = z[i];
          }
        }
      }
      tc_fence_before();
      mbar_arrive(&s_empty[b]);             // S of this buffer has been read
      // V rows of a partly filled last page hold pool bytes past k_cur, and the rows below
      // lo (the pages before soff and the first live page's slots before it, Q23*) bytes the
      // node no longer owns: zero them so that 0 · v stays 0 in Oᵀ = Vᵀ·Pᵀ (the rows past the
      // last page were zeroed before).  V of this stage has landed (MMA2 needs it anyway; P
      // is only published after)
      const int sv = k % NSV;
      mbar_wait(&full_v[sv][grp], (k / LV) & 1u);
      const int hi = span_hi(nt), lo = span_lo(nt);
      if (present && ((hi & (P - 1)) || lo)) {
        const int r0 = hi, r1 = (hi + P - 1) & ~(P - 1);
        unsigned char *Vs = Vst(sv);
        const int tl = trow - half * 64;   // 0..63 within the half
        for (int idx = tl; idx < (r1 - r0 + lo) * 16; idx += 64) {
          const int rr = idx >> 4;
          const int r = half * kHalf + (rr < lo ? rr : r0 + rr - lo), c16 = idx & 15;
          *reinterpret_cast<uint4 *>(Vs + (c16 >> 3) * 16384 + r * 128 + (c16 & 7) * 16) =
              make_uint4(0, 0, 0, 0);
        }
      }
      fence_proxy_async();
      named_bar_sync(bar_id, 128);
      mbar_arrive(&p_full[b]);
      if (tid == 64) TC_TRACE(k, 9);
    }
  } else {
    // ------------------------------------------------------------- epilogue (warps 6..9)
    // Oᵀ[d][n] (TMEM lane = d) → partials[pair A][li][h][g][d], in GW-column groups; the
    // tile's (m, l) per column after the four quadrants' max / sums
    constexpr int GW = kW<NQ>;
    const int quad = warp & 3;
    const int trow = quad * 32 + lane;
    const int G = a.G;
    const uint32_t lane_addr = static_cast<uint32_t>(quad * 32) << 16;
    const int SP = a.Lc * a.g.H * G;
    const int etid = tid - 192;                // 0..127
    for (int k = 0; k < ntiles; ++k) {
      const int b = k % kGroups;
      mbar_wait(&o_full[b], (k / kGroups) & 1u);
      if (tid == 192) TC_TRACE(k, 10);
      tc_fence_after();
      const TcHdr hd = ohdr[k % kHdrRing];   // read before o_empty (see the softmax)
      // m (log2 domain) and l of column n = etid, from the softmax ring slot k % kHdrRing
      float mm = 0.f, ll = 0.f;
      if (etid < NQ) {
        mm = fmaxf(fmaxf(red_m[k % kHdrRing][0][etid], red_m[k % kHdrRing][1][etid]),
                   fmaxf(red_m[k % kHdrRing][2][etid], red_m[k % kHdrRing][3][etid]));
        ll = (red_l[k % kHdrRing][0][etid] + red_l[k % kHdrRing][1][etid]) +
             (red_l[k % kHdrRing][2][etid] + red_l[k % kHdrRing][3][etid]);
      }
      const int qw = a.qw;
      const int ngrp = (min(NQ, qw * hd.cnt) + GW - 1) / GW;
      // columns of leaf slot j < cntA belong to pair A's group; a packed B half's columns
      // (slots cntA..cnt−1) to pair B's group
      const int cntA = hd.meta >> 4;
      const bool pack = (hd.meta & 2) != 0;
      const unsigned long long cm = pack ? colmask(cntA, G, qw) | (colmask(hd.cnt - cntA, G, qw) << (qw * cntA))
                                         : colmask(cntA, G, qw);
      float *pa = a.partials + ((static_cast<int64_t>(hd.pbA) * a.Lc + hd.li) * a.g.H + hd.h) * G * 130 + trow;
      float *pbq = a.partials + ((static_cast<int64_t>(pack ? hd.pbB : hd.pbA) * a.Lc + hd.li) * a.g.H + hd.h) * G * 130 + trow -
                   static_cast<int64_t>(cntA) * SP * 130;     // so that slot j ≥ cntA lands at j − cntA
      auto col_ptr = [&](int n) {
        return (col_j[n] < cntA ? pa : pbq) + static_cast<int64_t>(col_js[n]) * 130;
      };
#pragma unroll 1
      for (int gi = 0; gi < ngrp; ++gi) {
        const int c = gi * GW;
        float o[GW];
        tmem_ldW<GW>(tmem + lane_addr + b * 2 * NQ + NQ + c, o);
#pragma unroll
        for (int i = 0; i < GW; ++i) {
          const int n = c + i;
          if ((cm >> n) & 1ull) *col_ptr(n) = o[i];
        }
      }
      tc_fence_before();
      mbar_arrive(&o_empty[b]);
      if (etid < NQ && ((cm >> etid) & 1ull)) {
        float *dst = col_ptr(etid) - trow;
        dst[128] = mm;
        dst[129] = ll;
      }
      if (tid == 192) TC_TRACE(k, 11);
    }
  }
  tc_fence_before();
  __syncthreads();
  if (kTcTrace && a.trace && threadIdx.x == 0) {
    unsigned long long g1;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(g1));
    a.trace[(static_cast<int64_t>(blockIdx.x) * 64 + 63) * 16 + 1] = static_cast<long long>(g1);
    a.trace[(static_cast<int64_t>(blockIdx.x) * 64 + 63) * 16 + 2] = clock64() - t_start;
  }
  if (warp == 1) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;\n" ::"r"(tmem),
                 "r"(tmem_cols<NQ>()));
  }
}

template <int NQ, int NSK, int NSV>
void launch_tc(arbor_ctx *c, const TcArgs &a) {
  using S = TcSmem<NQ, NSK, NSV>;
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(attn_tc_kernel<NQ, NSK, NSV>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         static_cast<int>(S::kAlloc));
    attr = true;
  }
  static int sms = 0;
  if (!sms && cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0) != cudaSuccess) sms = 148;
  const int total = a.T * a.Lc * a.g.H;
  const int grid = total < sms ? total : sms;
  launch_pdl(attn_tc_kernel<NQ, NSK, NSV>, dim3(grid), dim3(kTcThreads), S::kAlloc, c->ms,
             *reinterpret_cast<const CUtensorMap *>(c->tmap_k),
             *reinterpret_cast<const CUtensorMap *>(c->tmap_v),
             *reinterpret_cast<const CUtensorMap *>(c->tmap_k4),
             *reinterpret_cast<const CUtensorMap *>(c->tmap_v4),
             *reinterpret_cast<const CUtensorMap *>(c->tmap_q[c->tmap_q_cur]), a);
}

long long *g_tc_trace = nullptr;

using EncodeTiledFn = CUresult (*)(CUtensorMap *, CUtensorMapDataType, cuuint32_t, void *,
                                   const cuuint64_t *, const cuuint64_t *, const cuuint32_t *,
                                   const cuuint32_t *, CUtensorMapInterleave, CUtensorMapSwizzle,
                                   CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
EncodeTiledFn g_encode = nullptr;

// [rows][128] bf16 viewed 2-D, box 64 × box_rows, SWIZZLE_128B (out-of-range rows read as 0)
bool encode_rows(void *map, const void *base, unsigned long long rows, unsigned box_rows) {
  const cuuint64_t dims[2] = {128, rows};
  const cuuint64_t strides[1] = {256};
  const cuuint32_t box[2] = {64, box_rows};
  const cuuint32_t es[2] = {1, 1};
  return g_encode(reinterpret_cast<CUtensorMap *>(map), CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2,
                  const_cast<void *>(base), dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                  CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                  CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

// The pool [L·NP][H][P][128] as 5-D (d-low 64, d-half 2, slot P, head H, layer·page L·NP),
// box {64, 1, P, 1, 64/P}: the 64 rows of 64/P consecutive pages of one (layer, head) and one
// d-half, landing as 64 consecutive 128-B swizzled rows (the K-major operand layout).
bool encode_pool5(void *map, const void *base, int L, int NP, int H, int P) {
  const cuuint64_t dims[5] = {64, 2, static_cast<cuuint64_t>(P), static_cast<cuuint64_t>(H),
                              static_cast<cuuint64_t>(L) * NP};
  const cuuint64_t strides[4] = {128, 256, static_cast<cuuint64_t>(P) * 256,
                                 static_cast<cuuint64_t>(H) * P * 256};
  const cuuint32_t box[5] = {64, 1, static_cast<cuuint32_t>(P), 1, static_cast<cuuint32_t>(64 / P)};
  const cuuint32_t es[5] = {1, 1, 1, 1, 1};
  return g_encode(reinterpret_cast<CUtensorMap *>(map), CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 5,
                  const_cast<void *>(base), dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                  CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                  CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

}  // namespace

// Tensor maps over the caller's K / V pools viewed as [rows = L·NP·H·P][d] bf16, box 64 × P,
// SWIZZLE_128B.  Returns false (the CUDA-core kernel is used) when the shape does not fit the
// tensor-core path or the driver entry point is unavailable.
bool attn_tc_init(arbor_ctx *c) {
  c->tc_ok = false;
  if (const char *e = getenv("ARBOR_ATTN")) {
    if (e[0] == 'c') return false;   // ARBOR_ATTN=cuda: force the CUDA-core kernel
  }
  if (c->esize != 2 || c->D != 128 || c->P % 16 != 0 || c->P > 64 || c->G > 8) return false;
  static_assert(sizeof(CUtensorMap) <= sizeof(c->tmap_k), "tensor map storage");
  if (!g_encode) {
    void *fn = nullptr;
    cudaDriverEntryPointQueryResult q{};
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q) != cudaSuccess ||
        q != cudaDriverEntryPointSuccess || !fn)
      return false;
    g_encode = reinterpret_cast<EncodeTiledFn>(fn);
  }
  const unsigned long long rows = static_cast<unsigned long long>(c->L) * c->NP * c->H * c->P;
  if (!encode_rows(c->tmap_k, c->cfg.k_pool, rows, static_cast<unsigned>(c->P)) ||
      !encode_rows(c->tmap_v, c->cfg.v_pool, rows, static_cast<unsigned>(c->P)) ||
      !encode_pool5(c->tmap_k4, c->cfg.k_pool, c->L, c->NP, c->H, c->P) ||
      !encode_pool5(c->tmap_v4, c->cfg.v_pool, c->L, c->NP, c->H, c->P))
    return false;
  c->tc_ok = true;
  return true;
}

// Launch the tensor-core attention if it applies to this plan; false → use the CUDA-core kernel.
bool launch_attn_tc(arbor_ctx *c, const PlanView &pv, const void *q, int layer_begin,
                    int layer_count, int max_cnt, void *out, float *lse) {
  if (!c->tc_ok || pv.T == 0) return false;
  // query slot rows per leaf: G (dense; the default) or 8 (ARBOR_QSLOT=8)
  static const int qslot8 = getenv("ARBOR_QSLOT") && atoi(getenv("ARBOR_QSLOT")) == 8;
  const int qw = qslot8 ? 8 : c->G;
  const int nq = qw * max_cnt;
  // q as [nA · layer_count · Hq rows][128]; re-encoded only when the buffer or its rows change
  const long long qrows = static_cast<long long>(pv.nA) * layer_count * c->Hq;
  int slot = -1;   // small cache of q tensor maps keyed by (buffer, rows)
  for (int i = 0; i < kQMaps; ++i)
    if (c->tmap_q_ptr[i] == q && c->tmap_q_rows[i] == qrows && c->tmap_q_box[i] == qw) slot = i;
  if (slot < 0) {
    slot = c->tmap_q_next;
    c->tmap_q_next = (c->tmap_q_next + 1) % kQMaps;
    if (!encode_rows(c->tmap_q[slot], q, static_cast<unsigned long long>(qrows),
                     static_cast<unsigned>(qw))) return false;
    c->tmap_q_ptr[slot] = q;
    c->tmap_q_rows[slot] = qrows;
    c->tmap_q_box[slot] = qw;
  }
  c->tmap_q_cur = slot;
  TcArgs a{};
  a.pv = pv;
  a.g = PoolView{c->L, c->H, c->P, c->D, c->NP, c->max_pages_node, c->max_tokens};
  a.ptab = c->d.ptab;
  a.kcur = c->d.kcur;
  a.soff = c->d.soff;
  a.q = static_cast<const __nv_bfloat16 *>(q);
  a.partials = c->d.partials;
  a.zbuf = c->d.zbuf;
  a.out = static_cast<__nv_bfloat16 *>(out);
  a.lse = lse;
  a.row_done = c->d.row_done;
  a.layer_begin = layer_begin;
  a.Lc = layer_count;
  a.Hq = c->Hq;
  a.G = c->G;
  a.T = pv.T;
  a.scale_log2 = kLog2e / sqrtf(128.f);
  a.qw = qw;
  static long long *trace = nullptr;
  if (getenv("ARBOR_TC_TRACE")) {
    if (!trace) cudaMalloc(&trace, sizeof(long long) * 148 * 64 * 16);
    cudaMemsetAsync(trace, 0, sizeof(long long) * 148 * 64 * 16, c->ms);
    a.trace = trace;
    g_tc_trace = trace;
  }
  // (K, V) ring depths; (4, 2) for NQ = 8 / 16 measured the same as (3, 3) on C2
  // NQ = 8 (single-leaf tiles: C2, C4, C5): two K / V stages — fewer bytes requested per SM at
  // the kernel start, the first tile lands sooner (round 2, late: attention +3.5-4.5% GB/s on
  // C2 / C4 / C5; -DARBOR_TC_NQ8_STAGES3 restores three)
#if defined(ARBOR_TC_NQ8_STAGES3)
  if (nq <= 8) launch_tc<8, 3, 3>(c, a);
#else
  if (nq <= 8) launch_tc<8, 2, 2>(c, a);
#endif
  else if (nq <= 16) launch_tc<16, 3, 3>(c, a);
  // NQ = 32 (the C3 frontier's 4-6-leaf tiles): three K stages, two V (round 2, late: C3
  // DPTS decode attention 156.3 -> 154.5 us once the trace code left the production build;
  // three V stages or 2 / 2 measured slower)
#if defined(ARBOR_TC_NQ32_NSK2)
  else if (nq <= 32) launch_tc<32, 2, 2>(c, a);
#elif defined(ARBOR_TC_NQ32_NSV3)
  else if (nq <= 32) launch_tc<32, 2, 3>(c, a);
#else
  else if (nq <= 32) launch_tc<32, 3, 2>(c, a);
#endif
  else if (nq <= 48) launch_tc<48, 2, 2>(c, a);
  else return false;
  return true;
}

}  // namespace arbor

// debug only (not part of include/arbor.h): copy the last ARBOR_TC_TRACE timeline to the host
extern "C" int arbor_debug_tc_trace(long long *host, long long count) {
  if (!arbor::g_tc_trace) return -1;
  cudaDeviceSynchronize();
  return cudaMemcpy(host, arbor::g_tc_trace, sizeof(long long) * count, cudaMemcpyDeviceToHost) == cudaSuccess ? 0 : -2;
}
