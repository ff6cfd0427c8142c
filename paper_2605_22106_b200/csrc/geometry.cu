// geometry.cu — §8(a) a1: depth d_i, Path*, Δ_i and the pinned set on the device.
//
// PAPER.md §3 Preliminaries: d_i = depth (root 0); Δ_i = shortest-path distance
// from i to the active leaf ℓ*; Path* = root→ℓ* chain.  With several active leaves
// (DPTS frontier) Path* is the union of chains and Δ_i the minimum distance (Q14).
// Pinned = Path* ∪ open blocks (invariant (i) P:104 read as k_i = n_i, Q19).
//
// One CTA; the tree is a few hundred to a few thousand nodes.  dist(i,ℓ) uses the LCA
// found by walking parent pointers (parent id < child id is validated on the host).
#include "common.cuh"

namespace arbor {
namespace {

__global__ void __launch_bounds__(1024)
geometry_kernel(int N, int nA, const int32_t *__restrict__ parent,
                const int32_t *__restrict__ active, const uint8_t *__restrict__ open,
                int32_t *__restrict__ depth, int32_t *__restrict__ delta,
                uint8_t *__restrict__ onpath, uint8_t *__restrict__ pinned, int k_protect) {
  // depth by walking to the root
  for (int i = threadIdx.x; i < N; i += blockDim.x) {
    int d = 0;
    for (int x = parent[i]; x >= 0; x = parent[x]) ++d;
    depth[i] = d;
    onpath[i] = 0;
  }
  __syncthreads();
  // Path* = ∪ Path(ℓ)
  for (int b = threadIdx.x; b < nA; b += blockDim.x) {
    for (int x = active[b]; x >= 0; x = parent[x]) onpath[x] = 1;
  }
  __syncthreads();
  // Δ_i = min_ℓ d_i + d_ℓ − 2 d_lca(i, ℓ)
  for (int i = threadIdx.x; i < N; i += blockDim.x) {
    int best = 0x7fffffff;
    const int di = depth[i];
    for (int b = 0; b < nA; ++b) {
      int x = i, y = active[b];
      int dx = di, dy = depth[y];
      while (dx > dy) { x = parent[x]; --dx; }
      while (dy > dx) { y = parent[y]; --dy; }
      while (x != y) { x = parent[x]; y = parent[y]; --dx; }
      const int dist = di + depth[active[b]] - 2 * dx;
      best = dist < best ? dist : best;
    }
    delta[i] = best;
    pinned[i] = ((onpath[i] && k_protect == 0) || open[i]) ? 1 : 0;   // P:104, Q19 (+STREAM)
  }
}

}  // namespace

void launch_geometry(arbor_ctx *c, int N, int nA) {
  stage_begin(c, ARBOR_ST_GEOMETRY, c->ms);
  geometry_kernel<<<1, 1024, 0, c->ms>>>(N, nA, c->d.parent, c->d.active, c->d.open,
                                          c->d.depth, c->d.delta, c->d.onpath, c->d.pinned,
                                          c->prm.alloc_mode == ARBOR_ALLOC_STREAM ? 1 : c->prm.k_protect);
  ARBOR_LAUNCHED(c);
  stage_end(c, ARBOR_ST_GEOMETRY, c->ms);
}

}  // namespace arbor
