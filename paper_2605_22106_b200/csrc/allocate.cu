// allocate.cu — §8(a) a4: Tree-Aware Eviction budget allocation on one CTA.
//
// PAPER.md §4 TAE: Eq. 2 r_i = clip(α η^{𝟙(i∉Path*)} s_i^γ e^{−λ_d d_i} e^{−λ_Δ Δ_i}, r_min, 1)
// (P:150-154); Eq. 3 k_i = min{n_i, max(K_min, |𝒯_i|, ⌊r_i n_i⌋)}; the
// optimisation view min Σ −w_i log k_i s.t. Σ k_i ≤ 𝓑, KKT k*_i = min{n_i, w_i/λ}
// (P:208-239); Alg. 2 Pressure drain.
//
// Exactness contract (Q9, Q10, Q12, Q29): the only floating point is one left-to-right fp64
// product per node with host-libm tables for the exp factors (no FMA contraction: __dmul_rn /
// __dadd_rn), W = round-half-even(w·2^24) as int64; everything after is integer:
//   WATERFILL: find λ with Σ clamp(W_j/λ, f_j, n_j) = 𝓑' by testing every breakpoint
//   W_j/n_j, W_j/f_j (one thread per candidate, 128-bit cross-multiplied sums), classify the
//   interval above the largest feasible breakpoint, k*_j = W_j·Num/Den on the active set,
//   then floor + largest remainder (ties: larger W, then smaller id) so Σ k = 𝓑 exactly.
//   STATIC: Eqs. 2-3 with the ε-floor.  STATIC_DRAIN: STATIC then the unit-step drain in
//   Priority order (W ascending, larger id first), done as one prefix sum.
#include "common.cuh"

namespace arbor {
namespace {

#ifndef ARBOR_ALLOC_THREADS
#define ARBOR_ALLOC_THREADS 512
#endif
constexpr int kThreads = ARBOR_ALLOC_THREADS;
constexpr double kWeightScale = 16777216.0;   // 2^24
constexpr double kEps = 1e-9;

struct AllocArgs {
  int N, Mpad;   // Mpad: breakpoint capacity (2N)
  long long budget;
  int mode;
  double alpha, gamma, eta, r_min;
  int k_min, l_tail, gamma_int;   // gamma_int ≥ 0: integer exponent (repeated products)
  int k_protect;                  // 0 → Path* pinned at n; > 0 → Path* floor min(n, k_protect)
  int n_sinks;                    // STREAM: the root's sink tokens
  const float *s;
  const int32_t *n;
  const int32_t *parent, *active;
  int nA;
  const uint8_t *open;
  uint8_t *onpath, *pinned;     // written (a1 fused)
  int32_t *depth, *delta;       // written (a1 fused)
  const double *Ed, *ED;
  int32_t *k_out;
  int only_node;   // ≥ 0: only this node's target is computed; the others get n (no change)
  const int32_t *gate;   // f1 device waterline: when *gate == 0, k_out = k_cur (no change)
  const int32_t *kcur;
  Ctrl *ctrl;
  long long *trace; // ARBOR_ALLOC_TRACE builds only: clock64() at phase boundaries
};

__device__ __forceinline__ int eps_floor_count(double r, int n) {
  // ⌊r·n + 1e-9⌋ (Q10), no contraction
  return static_cast<int>(floor(__dadd_rn(__dmul_rn(r, static_cast<double>(n)), kEps)));
}

__device__ __forceinline__ int keep_count(double r, int n, int k_min, int l_tail) {
  const int tl = min(l_tail, n);
  return min(n, max(max(k_min, tl), eps_floor_count(r, n)));
}

template <typename T>
__device__ T block_sum(T v, T *red) {
  // warp shuffle tree → one value per warp → warp 0 reduces → broadcast through red[0]
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5, nw = blockDim.x >> 5;
#pragma unroll
  for (int o = 16; o; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  __syncthreads();
  if (lane == 0) red[w] = v;
  __syncthreads();
  if (w == 0) {
    T x = lane < nw ? red[lane] : T(0);
#pragma unroll
    for (int o = 16; o; o >>= 1) x += __shfl_xor_sync(0xffffffffu, x, o);
    if (lane == 0) red[32] = x;
  }
  __syncthreads();
  return red[32];
}

// K integer block sums in one pass (three barriers instead of 3·K); exact, order-free
template <int K>
__device__ void block_sum_k(long long (&v)[K], long long (*red)[K]) {
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5, nw = blockDim.x >> 5;
#pragma unroll
  for (int k = 0; k < K; ++k)
#pragma unroll
    for (int o = 16; o; o >>= 1) v[k] += __shfl_xor_sync(0xffffffffu, v[k], o);
  __syncthreads();
  if (lane == 0)
#pragma unroll
    for (int k = 0; k < K; ++k) red[w][k] = v[k];
  __syncthreads();
  if (w == 0) {
#pragma unroll
    for (int k = 0; k < K; ++k) {
      long long x = lane < nw ? red[lane][k] : 0ll;
#pragma unroll
      for (int o = 16; o; o >>= 1) x += __shfl_xor_sync(0xffffffffu, x, o);
      if (lane == 0) red[32][k] = x;
    }
  }
  __syncthreads();
#pragma unroll
  for (int k = 0; k < K; ++k) v[k] = red[32][k];
}

// floor(X / den) and X mod den for 0 ≤ X < 2^126, 0 < den < 2^62, with a small quotient
__device__ __forceinline__ void divmod128(unsigned __int128 X, unsigned long long den,
                                          unsigned long long &q, unsigned long long &r) {
  unsigned long long qe = static_cast<unsigned long long>(
      static_cast<double>(X) / static_cast<double>(den));
  unsigned __int128 p = static_cast<unsigned __int128>(qe) * den;
  while (p > X) { --qe; p -= den; }
  while (p + den <= X) { ++qe; p += den; }
  q = qe;
  r = static_cast<unsigned long long>(X - p);
}

#ifdef ARBOR_ALLOC_TRACE
#define TRACE(i) do { if (threadIdx.x == 0 && a.trace) a.trace[i] = clock64(); } while (0)
#else
#define TRACE(i) do { } while (0)
#endif

__global__ void __launch_bounds__(kThreads)
allocate_kernel(AllocArgs a) {
  TRACE(0);
  extern __shared__ __align__(16) unsigned char sm[];
  const int N = a.N;
  long long *W = reinterpret_cast<long long *>(sm);            // [N]
  long long *rem = W + N;                                       // [N]
  int *nn = reinterpret_cast<int *>(rem + N);                   // [N]
  int *f = nn + N;                                              // [N]
  int *k = f + N;                                               // [N]
  int *cls = k + N;                                             // [N] class
  // breakpoint candidates (num int64 | den int32), 8-byte aligned; reused as rank[] later
  int *cand = cls + N;   // byte offset 32N: 8-byte aligned (the int64 candidate numerators)
  const int Mpad = a.Mpad;
  __shared__ long long red64[33];
  __shared__ unsigned long long best_num, best_den;
  __shared__ int best_set;

  // ---- a1 geometry (Alg. 2; Q14), fused: parent pointers in smem; depth by
  // walking to the root, Path* = ∪ root→ℓ chains, Δ_i = min_ℓ d_i + d_ℓ − 2·d_lca(i, ℓ).
  // Results also go to global memory (depth, Δ, Path*, pinned) for arbor_evict.  The tree
  // (parent, active) is uploaded by a copy before any kernel of the call, so the walks run
  // before griddepcontrol.wait and overlap the previous kernel's tail; the global writes
  // (which an earlier evict may still be reading) and every other read come after it.
  int *par = reinterpret_cast<int *>(cand + 3 * a.Mpad);         // [N] (after the candidates)
  int *dep = par + N;                                            // [N]
  int *dlt = dep + N;                                            // [N]
  int *act = dlt + N;                                            // [nA]
  unsigned char *onp = reinterpret_cast<unsigned char *>(act + a.nA);   // [N]
  for (int j = threadIdx.x; j < N; j += blockDim.x) {
    par[j] = a.parent[j];
    onp[j] = 0;
    dlt[j] = 0x7fffffff;
  }
  for (int b = threadIdx.x; b < a.nA; b += blockDim.x) act[b] = a.active[b];
  __syncthreads();
  for (int j = threadIdx.x; j < N; j += blockDim.x) {
    int d = 0;
    for (int x = par[j]; x >= 0; x = par[x]) ++d;
    dep[j] = d;
  }
  for (int b = threadIdx.x; b < a.nA; b += blockDim.x)
    for (int x = act[b]; x >= 0; x = par[x]) onp[x] = 1;
  __syncthreads();
  // one (node, active leaf) pair per thread — the LCA walks are dependent shared-memory
  // chains, so spreading the pairs (not the nodes) over the threads shortens the longest
  // chain nA-fold when nA is large (C3: 16 leaves); min over the leaves by shared atomics
  for (int u = threadIdx.x; u < N * a.nA; u += blockDim.x) {
    const int i = u / a.nA, b = u - i * a.nA;
    const int di = dep[i];
    int x = i, y = act[b];
    int dx = di, dy = dep[y];
    while (dx > dy) { x = par[x]; --dx; }
    while (dy > dx) { y = par[y]; --dy; }
    while (x != y) { x = par[x]; y = par[y]; --dx; }
    const int dist = di + dep[act[b]] - 2 * dx;
    if (a.nA == 1) dlt[i] = dist;     // one leaf: thread u owns node u (read back by it below)
    else atomicMin(&dlt[i], dist);
  }
  if (a.nA > 1) __syncthreads();
  pdl_wait();
  pdl_trigger();
  TRACE(3);
  if (a.gate && *a.gate == 0) {   // the waterline did not fire: no Pressure (Alg. 2 l.31-33)
    for (int i = threadIdx.x; i < N; i += blockDim.x) a.k_out[i] = a.kcur[i];
    return;
  }
  for (int i = threadIdx.x; i < N; i += blockDim.x) {
    a.depth[i] = dep[i];
    a.delta[i] = dlt[i];
    a.onpath[i] = onp[i];
    a.pinned[i] = ((onp[i] && a.k_protect == 0 && a.mode != 3) || a.open[i]) ? 1 : 0;
  }
  __syncthreads();

  // per-node weight, floors, pinned
  for (int j = threadIdx.x; j < N; j += blockDim.x) {
    const int nj = a.n[j];
    nn[j] = nj;
    // mode 3 (STREAM, the flattened-stream analogue): the path is a stream, not pinned
    const bool pin = (onp[j] && a.k_protect == 0 && a.mode != 3) || a.open[j];
    // protected Path* block: allocated like the others above min(n, k_protect)
    const int pf = (onp[j] && a.k_protect > 0) ? min(nj, a.k_protect) : 0;
    // w = s^γ · E_d[d] · E_Δ[Δ] · (η if off-path), strictly left to right
    const double s = static_cast<double>(a.s[j]);
    double w;
    if (a.gamma_int >= 0) {
      w = 1.0;
      for (int i = 0; i < a.gamma_int; ++i) w = __dmul_rn(w, s);
    } else {
      w = s > 0.0 ? exp(a.gamma * log(s)) : 0.0;
    }
    w = __dmul_rn(w, a.Ed[dep[j]]);
    w = __dmul_rn(w, a.ED[dlt[j]]);
    if (!onp[j]) w = __dmul_rn(w, a.eta);
    if (!(w >= 0.0) || w > 65536.0) {
      atomicOr(&a.ctrl->err, DERR_INVARIANT);
      w = 0.0;
    }
    W[j] = __double2ll_rn(__dmul_rn(w, kWeightScale));   // round-half-even(w·2^24)
    const int tl = min(a.l_tail, nj);
    f[j] = max(pf, min(nj, max(max(a.k_min, tl), eps_floor_count(a.r_min, nj))));
    if (pin) {
      k[j] = nj;
      cls[j] = 0;   // pinned
    } else if (a.mode == 3) {
      k[j] = 0;      // outside the stream until the path walk below
      cls[j] = 1;
    } else if (a.mode != 0) {
      // Eq. 2-3 (STATIC): r = clip(α·w, r_min, 1)
      const double r = fmin(1.0, fmax(a.r_min, __dmul_rn(a.alpha, w)));
      k[j] = max(pf, keep_count(r, nj, a.k_min, a.l_tail));
      cls[j] = 1;
    } else {
      k[j] = nj;
      cls[j] = W[j] > 0 ? 1 : 2;   // 1 = positive weight (P), 2 = zero weight (Z)
    }
  }
  __syncthreads();
  TRACE(1);

  if (a.mode == 2) {
    // STATIC_DRAIN: while Σk > 𝓑: j = argmin Priority (W asc, larger id first) over
    // non-pinned nodes with k > K_min; k_j ← max(K_min, k_j − 1)   (Alg. 2, Q16)
    long long tot = 0;
    for (int j = threadIdx.x; j < N; j += blockDim.x) tot += k[j];
    tot = block_sum(tot, red64);
    long long excess = tot - a.budget;
    // drain floor of node j: K_min (Alg. 2), raised to min(n, k_protect) on a
    // protected Path* block
    auto dfl = [&](int j) {
      return (onp[j] && a.k_protect > 0) ? max(a.k_min, min(nn[j], a.k_protect)) : a.k_min;
    };
    if (excess > 0) {
      // rank of each drainable node in priority order (stored in f[], floors are unused in
      // this mode); capacity k_j − K_min into rem[rank]
      for (int j = threadIdx.x; j < N; j += blockDim.x) rem[j] = 0;
      __syncthreads();
      for (int j = threadIdx.x; j < N; j += blockDim.x) {
        int rank = -1;
        if (cls[j] == 1 && k[j] > dfl(j)) {
          rank = 0;
          for (int i = 0; i < N; ++i) {
            if (cls[i] == 1 && k[i] > dfl(i) &&
                (W[i] < W[j] || (W[i] == W[j] && i > j)))
              ++rank;
          }
        }
        f[j] = rank;
      }
      __syncthreads();
      for (int j = threadIdx.x; j < N; j += blockDim.x)
        if (f[j] >= 0) rem[f[j]] = k[j] - dfl(j);
      __syncthreads();
      if (threadIdx.x == 0) {   // exclusive prefix over ranks (N ≤ 4096, serial is fine)
        long long acc = 0;
        for (int r = 0; r < N; ++r) {
          const long long c = rem[r];
          rem[r] = acc;
          acc += c;
        }
      }
      __syncthreads();
      for (int j = threadIdx.x; j < N; j += blockDim.x) {
        if (f[j] >= 0) {
          const long long before = rem[f[j]];
          const long long cap = k[j] - dfl(j);
          long long dr = excess - before;
          dr = dr < 0 ? 0 : (dr > cap ? cap : dr);
          k[j] -= static_cast<int>(dr);
        }
      }
    }
  } else if (a.mode == 3) {
    // ---- STREAM: the sequence-flattened StreamingLLM analogue ----
    // the single active path root → ℓ keeps the root's first n_sinks tokens and its most
    // recent 𝓑 − Σ_open n − |sinks| tokens, walking from ℓ up (oracle/tae.stream_targets)
    long long open_n = 0;
    for (int j = threadIdx.x; j < N; j += blockDim.x) if (a.open[j]) open_n += nn[j];
    open_n = block_sum(open_n, red64);
    if (threadIdx.x == 0) {
      const int s0 = a.open[0] ? 0 : min(a.n_sinks, nn[0]);
      long long rem = a.budget - open_n - s0;   // ≥ 0: the host checked min_feasible
      for (int x = act[0]; x >= 0; x = par[x]) {
        if (a.open[x]) continue;
        const int w = static_cast<int>(min(static_cast<long long>(nn[x]), rem));
        rem -= w;
        k[x] = x == 0 ? min(nn[x], s0 + w) : w;
      }
    }
  } else if (a.mode == 0) {
    // ---- WATERFILL (optimisation view) ----
    long long T = 0, pinned_n = 0, free_n = 0, SnP = 0, SfZ = 0, SslZ = 0;
    for (int j = threadIdx.x; j < N; j += blockDim.x) {
      T += nn[j];
      if (cls[j] == 0) pinned_n += nn[j];
      else free_n += nn[j];
      if (cls[j] == 1) SnP += nn[j];
      if (cls[j] == 2) { SfZ += f[j]; SslZ += nn[j] - f[j]; }
    }
    {
      __shared__ long long red6[33][6];
      long long v6[6] = {T, pinned_n, free_n, SnP, SfZ, SslZ};
      block_sum_k<6>(v6, red6);
      T = v6[0]; pinned_n = v6[1]; free_n = v6[2]; SnP = v6[3]; SfZ = v6[4]; SslZ = v6[5];
    }
    TRACE(2);
    const long long Bp = a.budget - pinned_n;
    if (T <= a.budget || Bp >= free_n) {
      // full retention (k = n already)
    } else if (SnP + SfZ <= Bp) {
      // step 10: positive-weight nodes saturate; spread R over zero-weight nodes by slack
      const long long R = Bp - SnP - SfZ;
      long long given = 0;
      for (int j = threadIdx.x; j < N; j += blockDim.x) {
        if (cls[j] == 2) {
          const long long sl = nn[j] - f[j];
          const long long x = sl * R;
          const long long b = SslZ > 0 ? x / SslZ : 0;
          rem[j] = SslZ > 0 ? x % SslZ : 0;
          k[j] = f[j] + static_cast<int>(b);
          given += b;
        }
      }
      given = block_sum(given, red64);
      const long long leftover = R - given;
      for (int j = threadIdx.x; j < N; j += blockDim.x) {
        if (cls[j] == 2 && leftover > 0) {
          long long rank = 0;
          for (int i = 0; i < N; ++i)
            if (cls[i] == 2 && (rem[i] > rem[j] || (rem[i] == rem[j] && i < j))) ++rank;
          if (rank < leftover) k[j] += 1;
        }
      }
    } else {
      // zero-weight nodes keep their floor; waterfill the positive-weight nodes with 𝓑''
      for (int j = threadIdx.x; j < N; j += blockDim.x)
        if (cls[j] == 2) k[j] = f[j];
      const long long Bpp = Bp - SfZ;
      // S(λ) = Σ_j clamp(W_j/λ, f_j, n_j) is continuous and nonincreasing; its breakpoints
      // are W_j/n_j and W_j/f_j (f_j > 0).  β* = the largest breakpoint with S(β*) ≥ 𝓑''
      // (exact: S(β) ≥ 𝓑'' ⇔ SA·den ≥ (𝓑'' − Sb)·num in 128-bit, W < 2^40, n, f < 2^15).
      // Multisection: each round a warp per pivot tests 16 pivots exactly; the candidates
      // outside [largest feasible pivot, smallest infeasible pivot) are dropped; ≤ 16 left →
      // test them all.  ~3 rounds for a few hundred breakpoints.
      long long *cnum = reinterpret_cast<long long *>(cand);          // [2N]
      int *cden = reinterpret_cast<int *>(cnum + 2 * N);              // [2N]
      __shared__ int ncand, nnext, piv_ok[kThreads / 32];
      __shared__ long long lo_num, hi_num;
      __shared__ int lo_den, hi_den, lo_set, hi_set;
      if (threadIdx.x == 0) ncand = 0;
      __syncthreads();
      const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nw = blockDim.x >> 5;
      const unsigned lt = (1u << lane) - 1u;
      for (int c0 = 0; c0 < 2 * N; c0 += blockDim.x) {   // warp-aggregated append
        const int c = c0 + threadIdx.x;
        const int j = c >> 1;
        const bool take = c < 2 * N && cls[j] == 1 && ((c & 1) == 0 || f[j] > 0);
        const unsigned bal = __ballot_sync(0xffffffffu, take);
        int base = 0;
        if (lane == 0 && bal) base = atomicAdd(&ncand, __popc(bal));
        base = __shfl_sync(0xffffffffu, base, 0);
        if (take) {
          const int slot = base + __popc(bal & lt);
          cnum[slot] = W[j];
          cden[slot] = (c & 1) ? f[j] : nn[j];
        }
      }
      __syncthreads();
      // exact feasibility of β = num/den, one warp (lanes over nodes)
      auto feasible = [&](long long cn, long long cd) -> bool {
        long long SA = 0, Sb = 0;
        for (int i = lane; i < N; i += 32) {
          if (cls[i] != 1) continue;
          const long long Wd = W[i] * cd;
          const long long ni = nn[i], fi = f[i];
          if (Wd >= ni * cn) Sb += ni;                       // capped
          else if (fi > 0 && Wd <= fi * cn) Sb += fi;        // floored
          else SA += W[i];                                   // active
        }
        // warp sums with 32-bit reductions: per-lane SA < 2^48 split at bit 24, Sb < 2^30
        const unsigned lo = __reduce_add_sync(0xffffffffu, static_cast<unsigned>(SA & 0xFFFFFF));
        const unsigned hi = __reduce_add_sync(0xffffffffu, static_cast<unsigned>(SA >> 24));
        const unsigned sb = __reduce_add_sync(0xffffffffu, static_cast<unsigned>(Sb));
        const long long SAt = (static_cast<long long>(hi) << 24) + lo, Sbt = sb;
        return static_cast<__int128>(SAt) * cd >= static_cast<__int128>(Bpp - Sbt) * cn;
      };
      int M = ncand;
      int stall = 0;
#ifdef ARBOR_ALLOC_TRACE
      int rounds = 0;
      if (threadIdx.x == 0 && a.trace) a.trace[8] = ncand;
#endif
      while (M > 0) {
#ifdef ARBOR_ALLOC_TRACE
        ++rounds;
#endif
        const bool all = M <= nw || stall;   // test every remaining candidate this round
        const int P = all ? M : nw;
        // pivots: evenly spaced list entries (all entries when testing all)
        for (int p0 = 0; p0 < P; p0 += nw) {
          const int p = p0 + wid;
          if (p < P) {
            const int e = all ? p : static_cast<int>((static_cast<long long>(p) * M) / P);
            const bool ok = feasible(cnum[e], cden[e]);
            if (lane == 0) piv_ok[wid] = ok;
          }
          __syncthreads();
          if (wid == 0) {
            // lane w < P: pivot w; warp max over the feasible ratios, min over the infeasible
            const int pw = p0 + lane;
            const bool have = lane < nw && pw < P;
            long long cn = 0;
            int cd = 1, okf = 0;
            if (have) {
              const int e = all ? pw : static_cast<int>((static_cast<long long>(pw) * M) / P);
              cn = cnum[e];
              cd = cden[e];
              okf = piv_ok[lane];
            }
            long long ln = cn, hn = cn;
            int ld = cd, hd = cd;
            int ls = have && okf, hs = have && !okf;
            if (p0 > 0) {   // fold in the previous batch (lane 0 carries it)
              if (lane == 0 && lo_set && (!ls || lo_num * ld > ln * lo_den)) { ln = lo_num; ld = lo_den; ls = 1; }
              if (lane == 0 && hi_set && (!hs || hi_num * hd < hn * hi_den)) { hn = hi_num; hd = hi_den; hs = 1; }
            }
#pragma unroll
            for (int o = 16; o; o >>= 1) {
              const long long on = __shfl_xor_sync(0xffffffffu, ln, o);
              const int od = __shfl_xor_sync(0xffffffffu, ld, o), os = __shfl_xor_sync(0xffffffffu, ls, o);
              if (os && (!ls || on * ld > ln * od)) { ln = on; ld = od; ls = 1; }
              const long long hn2 = __shfl_xor_sync(0xffffffffu, hn, o);
              const int hd2 = __shfl_xor_sync(0xffffffffu, hd, o), hs2 = __shfl_xor_sync(0xffffffffu, hs, o);
              if (hs2 && (!hs || hn2 * hd < hn * hd2)) { hn = hn2; hd = hd2; hs = 1; }
            }
            if (lane == 0) {
              lo_num = ln; lo_den = ld; lo_set = ls;
              hi_num = hn; hi_den = hd; hi_set = hs;
            }
          }
          __syncthreads();
        }
        if (all) break;
        // keep lo ≤ ratio < hi (compacted in place: read all, then write)
        if (threadIdx.x == 0) nnext = 0;
        __syncthreads();
        constexpr int kCap = (2 * 3072 + kThreads - 1) / kThreads;   // max_nodes ≤ 3072
        long long kn[kCap];
        int kd[kCap], kc = 0;
        for (int e = threadIdx.x; e < M; e += blockDim.x) {
          const long long cn = cnum[e];
          const int cd = cden[e];
          const bool ge_lo = !lo_set || cn * lo_den >= lo_num * cd;
          const bool lt_hi = !hi_set || cn * hi_den < hi_num * cd;
          if (ge_lo && lt_hi) { kn[kc] = cn; kd[kc] = cd; ++kc; }
        }
        __syncthreads();
        const int base = kc ? atomicAdd(&nnext, kc) : 0;
        for (int i = 0; i < kc; ++i) { cnum[base + i] = kn[i]; cden[base + i] = kd[i]; }
        __syncthreads();
        stall = nnext == M;   // every pivot tied with lo: test all the rest next round
        M = nnext;
      }
      __syncthreads();
      if (threadIdx.x == 0) {
        if (!lo_set) {
          atomicOr(&a.ctrl->err, DERR_INVARIANT);
          best_num = 0;
          best_den = 1;
        } else {
          best_num = static_cast<unsigned long long>(lo_num);
          best_den = static_cast<unsigned long long>(lo_den);
        }
        best_set = 1;
      }
      __syncthreads();
      TRACE(4);
#ifdef ARBOR_ALLOC_TRACE
      if (threadIdx.x == 0 && a.trace) a.trace[7] = rounds;
#endif
      const long long bnum = static_cast<long long>(best_num);
      const long long bden = static_cast<long long>(best_den);
      // classify the open interval just above β
      long long Sb = 0, Den = 0;
      for (int j = threadIdx.x; j < N; j += blockDim.x) {
        if (cls[j] != 1) continue;
        const long long Wd = W[j] * bden;
        if (Wd > static_cast<long long>(nn[j]) * bnum) { k[j] = nn[j]; Sb += nn[j]; cls[j] = 4; }
        else if (f[j] > 0 && Wd <= static_cast<long long>(f[j]) * bnum) { k[j] = f[j]; Sb += f[j]; cls[j] = 5; }
        else { Den += W[j]; cls[j] = 6; }   // active
      }
      {
        __shared__ long long red2[33][2];
        long long v2[2] = {Sb, Den};
        block_sum_k<2>(v2, red2);
        Sb = v2[0];
        Den = v2[1];
      }
      const long long Num = Bpp - Sb;
      long long given = 0;
      for (int j = threadIdx.x; j < N; j += blockDim.x) {
        if (cls[j] != 6) continue;
        unsigned long long q = 0, r = 0;
        if (Num > 0 && Den > 0) {
          divmod128(static_cast<unsigned __int128>(W[j]) * static_cast<unsigned long long>(Num),
                    static_cast<unsigned long long>(Den), q, r);
        }
        k[j] = static_cast<int>(q);
        rem[j] = static_cast<long long>(r);
        given += static_cast<long long>(q);
      }
      given = block_sum(given, red64);
      TRACE(5);
      const long long leftover = Num - given;
#ifndef ARBOR_ALLOC_LR_WARP_MAX
#define ARBOR_ALLOC_LR_WARP_MAX 256   // trees up to this size rank by warp per node
#endif
      if (leftover > 0 && N <= ARBOR_ALLOC_LR_WARP_MAX) {
        // largest remainder: the `leftover` active nodes first in (rem desc, W desc, id asc)
        // get +1.  Small trees: rank of each active node — a warp per node, lanes over the
        // other nodes, one __reduce_add_sync per node (O(N²/32): 4.8 µs at N = 156)
        int *rank = cand;                       // the breakpoint list is no longer needed
        const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nw = blockDim.x >> 5;
        for (int j = wid; j < N; j += nw) {
          if (cls[j] != 6) continue;            // warp-uniform
          const long long rj = rem[j], Wj = W[j];
          unsigned cnt = 0;
          for (int i = lane; i < N; i += 32) {
            const long long ri = rem[i], Wi = W[i];
            cnt += (cls[i] == 6) & ((ri > rj) | ((ri == rj) & ((Wi > Wj) | ((Wi == Wj) & (i < j)))));
          }
          cnt = __reduce_add_sync(0xffffffffu, cnt);
          if (lane == 0) rank[j] = static_cast<int>(cnt);
        }
        __syncthreads();
        for (int j = threadIdx.x; j < N; j += blockDim.x)
          if (cls[j] == 6 && rank[j] < leftover) k[j] += 1;
      } else if (leftover > 0) {
        // larger trees: bitonic sort of the active ids in shared memory by the same key (keys
        // are unique — the id breaks every tie — so the compaction order does not matter);
        // the quadratic ranking took 23 µs at N = 512 (C5), this 15 µs
        int *idx = cand;
        __shared__ int na_s;
        if (threadIdx.x == 0) na_s = 0;
        __syncthreads();
        for (int j = threadIdx.x; j < N; j += blockDim.x)
          if (cls[j] == 6) idx[atomicAdd(&na_s, 1)] = j;
        __syncthreads();
        const int na = na_s;
        int P2 = 1;
        while (P2 < na) P2 <<= 1;
        for (int t = na + threadIdx.x; t < P2; t += blockDim.x) idx[t] = -1;   // sentinels: last
        __syncthreads();
        auto gt = [&](int x, int y) {           // key(x) > key(y); −1 below everything
          if (y < 0) return x >= 0;
          if (x < 0) return false;
          if (rem[x] != rem[y]) return rem[x] > rem[y];
          if (W[x] != W[y]) return W[x] > W[y];
          return x < y;
        };
#ifndef ARBOR_ALLOC_LR_SHFL
#define ARBOR_ALLOC_LR_SHFL 1
#endif
        if (ARBOR_ALLOC_LR_SHFL && P2 <= kThreads) {
          // ≤ 512 keys: one per thread, the key (rem, W, id) in registers; a compare-exchange
          // stage of stride < 32 is a warp shuffle, only strides ≥ 32 go through shared memory
          // with a barrier (10 barrier stages at 512 keys instead of 45)
          const int P = P2 < 64 ? 64 : P2;    // whole warps
          for (int t = na + threadIdx.x; t < P; t += blockDim.x) idx[t] = -1;
          __syncthreads();
          const int t = threadIdx.x;
          int x = t < P ? idx[t] : -1;
          long long xr = x >= 0 ? rem[x] : 0, xw = x >= 0 ? W[x] : 0;
          auto gtk = [](int a, long long ar, long long aw, int b, long long br, long long bw) {
            if (b < 0) return a >= 0;
            if (a < 0) return false;
            if (ar != br) return ar > br;
            if (aw != bw) return aw > bw;
            return a < b;
          };
          for (int size = 2; size <= P; size <<= 1) {
            for (int stride = size >> 1; stride > 0; stride >>= 1) {
              int y;
              long long yr, yw;
              if (stride >= 32) {
                __syncthreads();                 // the previous stage's reads are done
                if (t < P) idx[t] = x;
                __syncthreads();
                y = t < P ? idx[t ^ stride] : -1;
                yr = y >= 0 ? rem[y] : 0;
                yw = y >= 0 ? W[y] : 0;
              } else {
                y = __shfl_xor_sync(0xffffffffu, x, stride);
                yr = __shfl_xor_sync(0xffffffffu, xr, stride);
                yw = __shfl_xor_sync(0xffffffffu, xw, stride);
              }
              const bool lower = (t & stride) == 0, desc = (t & size) == 0;
              // a descending run keeps the larger key at the lower position
              const bool take = (lower == desc) ? gtk(y, yr, yw, x, xr, xw) : gtk(x, xr, xw, y, yr, yw);
              if (take) { x = y; xr = yr; xw = yw; }
            }
          }
          if (t < leftover && x >= 0) k[x] += 1;
        } else
        for (int size = 2; size <= P2; size <<= 1) {
          for (int stride = size >> 1; stride > 0; stride >>= 1) {
            for (int i = threadIdx.x; i < P2; i += blockDim.x) {
              const int p = i ^ stride;
              if (p > i) {
                const int x = idx[i], y = idx[p];
                const bool desc = (i & size) == 0;   // this run sorted descending
                if (desc ? gt(y, x) : gt(x, y)) { idx[i] = y; idx[p] = x; }
              }
            }
            __syncthreads();
          }
        }
        if (!(ARBOR_ALLOC_LR_SHFL && P2 <= kThreads))
          for (int t = threadIdx.x; t < leftover; t += blockDim.x) k[idx[t]] += 1;
      }
    }
  }
  __syncthreads();
  TRACE(6);
  for (int j = threadIdx.x; j < N; j += blockDim.x)
    a.k_out[j] = (a.only_node < 0 || j == a.only_node) ? k[j] : nn[j];
}

}  // namespace

__global__ void waterline_kernel(const int32_t *__restrict__ kcur, int N, long long thresh,
                                 int infeasible, Ctrl *ctrl) {
  __shared__ long long red[32];
  long long m = 0;
  for (int i = threadIdx.x; i < N; i += blockDim.x) m += kcur[i];
#pragma unroll
  for (int o = 16; o; o >>= 1) m += __shfl_xor_sync(0xffffffffu, m, o);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = m;
  __syncthreads();
  if (threadIdx.x == 0) {
    long long tot = 0;
    for (int w = 0; w < static_cast<int>(blockDim.x >> 5); ++w) tot += red[w];
    const int fire = tot >= thresh ? 1 : 0;     // M ≥ 𝓑 − δ (Alg. 2 l.31)
    ctrl->gate = infeasible ? 0 : fire;
    if (fire && infeasible) atomicOr(&ctrl->err, DERR_INFEASIBLE);
    if (fire && !infeasible) ctrl->pressure_events += 1;
  }
}

void launch_waterline(arbor_ctx *c, int N, int64_t thresh, bool infeasible) {
  waterline_kernel<<<1, 256, 0, c->ms>>>(c->d.kcur, N, thresh, infeasible ? 1 : 0, c->d.ctrl);
  ARBOR_LAUNCHED(c);
}

void launch_allocate(arbor_ctx *c, int N, int nA, const float *s, int64_t budget, int32_t *k_out,
                     int mode, int only_node, bool gated) {
  AllocArgs a{};
  a.gate = gated ? &c->d.ctrl->gate : nullptr;
  a.kcur = c->d.kcur;
  a.N = N;
  a.budget = budget;
  a.mode = mode < 0 ? c->prm.alloc_mode : mode;
  a.only_node = only_node;
  a.alpha = c->prm.alpha;
  a.gamma = c->prm.gamma;
  a.eta = c->prm.eta;
  a.r_min = c->prm.r_min;
  a.k_min = c->prm.k_min;
  a.l_tail = c->prm.l_tail;
  a.k_protect = c->prm.k_protect;
  a.n_sinks = c->prm.n_sinks;
  const double g = c->prm.gamma;
  a.gamma_int = (g >= 0.0 && g <= 64.0 && g == static_cast<double>(static_cast<int>(g)))
                    ? static_cast<int>(g) : -1;
  a.s = s;
  a.n = c->d.len;
  a.parent = c->d.parent;
  a.active = c->d.active;
  a.nA = nA;
  a.onpath = c->d.onpath;
  a.pinned = c->d.pinned;
  a.open = c->d.open;
  a.depth = c->d.depth;
  a.delta = c->d.delta;
  a.Ed = c->d.Ed;
  a.ED = c->d.ED;
  a.k_out = k_out;
  a.ctrl = c->d.ctrl;
  a.trace = c->d.alloc_trace;
  a.Mpad = 2 * N;
  // [W rem | nn f k cls | candidates (2N × 12 B, as 3·Mpad ints) | par dep dlt | act | onp]
  const size_t smem = static_cast<size_t>(N) * (2 * sizeof(long long) + 4 * sizeof(int)) + 8 +
                      static_cast<size_t>(3 * a.Mpad) * sizeof(int) +
                      static_cast<size_t>(3 * N + nA) * sizeof(int) + N + 16;
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(allocate_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 220 * 1024);
    attr = true;
  }
  stage_begin(c, ARBOR_ST_ALLOCATE, c->ms);
  launch_pdl(allocate_kernel, dim3(1), dim3(kThreads), smem, c->ms, a);
  ARBOR_LAUNCHED(c);
  stage_end(c, ARBOR_ST_ALLOCATE, c->ms);
}

}  // namespace arbor
