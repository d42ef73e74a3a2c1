// Grid-wide barrier for cooperative persistent kernels (co-residency is
// guaranteed by cudaLaunchCooperativeKernel).  Bounded spin: a barrier that
// waits ~seconds raises `abort` so a bug cannot wedge the GPU.
#pragma once
#include "common.cuh"

namespace pip {

struct GridSync {
  u32 bar_count, bar_gen, abort, error;
};

// ---------------------------------------------------------------------------
// grid barrier (co-residency guaranteed by the cooperative launch)
__device__ __forceinline__ bool grid_barrier(GridSync* g, u32& gen) {
  __syncthreads();
  __shared__ int s_ok;
  if (threadIdx.x == 0) {
    int ok = 1;
    __threadfence();
    const u32 arrived = atomicAdd(&g->bar_count, 1u);
    if (arrived == gridDim.x - 1) {
      atomicExch(&g->bar_count, 0u);
      __threadfence();
      st_release_u32(&g->bar_gen, gen + 1);
    } else {
      u64 spins = 0;
      while (ld_acquire_u32(&g->bar_gen) == gen) {
        if (++spins > 32) __nanosleep(32);
        if ((spins & 1023) == 0) {
          if (ld_relaxed_u32(&g->abort)) { ok = 0; break; }
          if (spins > (1ull << 26)) { atomicExch(&g->abort, 1u); ok = 0; break; }
        }
      }
    }
    gen += 1;
    __threadfence();
    s_ok = ok;
  }
  __syncthreads();
  // propagate gen to all threads (only thread 0 uses it, but keep uniform)
  return s_ok;
}

}  // namespace pip
