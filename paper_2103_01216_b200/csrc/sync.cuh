// Grid-wide barrier for cooperative persistent kernels (co-residency is
// guaranteed by cudaLaunchCooperativeKernel).  Bounded spin: a barrier that
// waits ~seconds raises `abort` so a bug cannot wedge the GPU.
#pragma once
#include "common.cuh"

namespace pip {

#ifndef PIP_BAR_SPIN
#define PIP_BAR_SPIN 16  // polls before the barrier waiter starts sleeping between polls
#endif

struct GridSync {
  u32 bar_count, bar_gen, abort, error;
};

// ---------------------------------------------------------------------------
// grid barrier (co-residency guaranteed by the cooperative launch).  The
// arrival counter only grows (barrier k of a launch completes when it reaches
// k * gridDim.x), so the last arriver has nothing to reset or publish: one
// acq_rel add per CTA, then acquire polls of the same word.  `bar_count` is
// zeroed before every launch.
__device__ __forceinline__ u32 atom_add_acq_rel_u32(u32* p, u32 v) {
  u32 old;
  asm volatile("atom.acq_rel.gpu.global.add.u32 %0, [%1], %2;" : "=r"(old) : "l"(p), "r"(v) : "memory");
  return old;
}

__device__ __forceinline__ bool grid_barrier(GridSync* g, u32& gen) {
  __syncthreads();
  __shared__ int s_ok;
  if (threadIdx.x == 0) {
    int ok = 1;
    const u32 target = (gen + 1) * gridDim.x;
    u32 v = atom_add_acq_rel_u32(&g->bar_count, 1u) + 1u;
    u64 spins = 0;
    while ((int)(v - target) < 0) {
      if (++spins > PIP_BAR_SPIN) __nanosleep(32);
      if ((spins & 1023) == 0) {
        if (ld_relaxed_u32(&g->abort)) { ok = 0; break; }
        if (spins > (1ull << 26)) { atomicExch(&g->abort, 1u); ok = 0; break; }
      }
      v = ld_acquire_u32(&g->bar_count);
    }
    gen += 1;
    s_ok = ok;
  }
  __syncthreads();
  return s_ok;
}

}  // namespace pip
