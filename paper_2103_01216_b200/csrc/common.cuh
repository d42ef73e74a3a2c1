// Shared device helpers for the PIP kernels (sm_100a).
#pragma once
#include <cstdint>
#include <cuda_runtime.h>
#include "../../include/pip.h"

typedef unsigned long long u64;
typedef unsigned int u32;

namespace pip {

// ---------------------------------------------------------------------------
// error plumbing (host)
void set_cuda_error(cudaError_t e);
#define PIP_CUDA(call)                                   \
  do {                                                   \
    cudaError_t _e = (call);                             \
    if (_e != cudaSuccess) {                             \
      ::pip::set_cuda_error(_e);                         \
      return PIP_ERR_CUDA;                               \
    }                                                    \
  } while (0)
#define PIP_CHECK_LAUNCH() PIP_CUDA(cudaGetLastError())

int num_sms(int device);
int current_device();

// ---------------------------------------------------------------------------
// memory-model helpers (PTX acquire / release at GPU scope)
__device__ __forceinline__ u32 ld_acquire_u32(const u32* p) {
  u32 v;
  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ u32 ld_relaxed_u32(const u32* p) {
  u32 v;
  asm volatile("ld.relaxed.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ u64 ld_relaxed_u64(const u64* p) {
  u64 v;
  asm volatile("ld.relaxed.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_release_u32(u32* p, u32 v) {
  asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ void st_relaxed_u32(u32* p, u32 v) {
  asm volatile("st.relaxed.gpu.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ void st_relaxed_u64(u64* p, u64 v) {
  asm volatile("st.relaxed.gpu.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ void fence_gpu() { asm volatile("fence.acq_rel.gpu;" ::: "memory"); }

// streaming (evict-first) global accesses for data touched exactly once
__device__ __forceinline__ ulonglong2 ldg_stream2(const u64* p) {
  ulonglong2 v;
  asm volatile("ld.global.cs.v2.u64 {%0, %1}, [%2];" : "=l"(v.x), "=l"(v.y) : "l"(p));
  return v;
}
__device__ __forceinline__ void stg_stream2(u64* p, u64 x, u64 y) {
  asm volatile("st.global.cs.v2.u64 [%0], {%1, %2};" ::"l"(p), "l"(x), "l"(y) : "memory");
}

// ---------------------------------------------------------------------------
// element operations (strong.scan's `op`; all associative and commutative)
template <int OP> struct Op;
template <> struct Op<PIP_OP_ADD> {
  static constexpr u64 identity = 0ull;
  __device__ __forceinline__ static u64 apply(u64 a, u64 b) { return a + b; }
};
template <> struct Op<PIP_OP_MAX> {
  static constexpr u64 identity = 0ull;
  __device__ __forceinline__ static u64 apply(u64 a, u64 b) { return a > b ? a : b; }
};
template <> struct Op<PIP_OP_MIN> {
  static constexpr u64 identity = ~0ull;
  __device__ __forceinline__ static u64 apply(u64 a, u64 b) { return a < b ? a : b; }
};
template <> struct Op<PIP_OP_XOR> {
  static constexpr u64 identity = 0ull;
  __device__ __forceinline__ static u64 apply(u64 a, u64 b) { return a ^ b; }
};

// ---------------------------------------------------------------------------
// predicate (pip_pred) with u64 magic-number division for MOD_EQ
struct DevPred {
  u32 kind, negate;
  u64 a, b;
  u64 magic;   // MOD_EQ: multiplier
  u32 shift;   // MOD_EQ: post shift
  u32 add;     // MOD_EQ: 65-bit "add" form
  u32 pow2;    // MOD_EQ: divisor is a power of two (use mask a-1)
};
DevPred make_dev_pred(const pip_pred& p);

__device__ __forceinline__ u64 fast_div(u64 x, const DevPred& p) {
  u64 q = __umul64hi(x, p.magic);
  if (p.add) {
    u64 t = ((x - q) >> 1) + q;
    return t >> p.shift;
  }
  return q >> p.shift;
}

__device__ __forceinline__ bool pred_eval(const DevPred& p, u64 x) {
  bool r;
  switch (p.kind) {
    case PIP_PRED_MASK_EQ: r = (x & p.a) == p.b; break;
    case PIP_PRED_MOD_EQ: {
      u64 m;
      if (p.pow2) m = x & (p.a - 1);
      else m = x - fast_div(x, p) * p.a;
      r = m == p.b;
      break;
    }
    case PIP_PRED_LT: r = x < p.a; break;
    case PIP_PRED_LE: r = x <= p.a; break;
    case PIP_PRED_GT: r = x > p.a; break;
    case PIP_PRED_GE: r = x >= p.a; break;
    case PIP_PRED_EQ: r = x == p.a; break;
    default: r = true; break;
  }
  return r != (p.negate != 0);
}

// ---------------------------------------------------------------------------
// runtime.Rng (SplitMix64 finalizer over a golden-ratio counter)
static constexpr u64 GOLDEN = 0x9E3779B97F4A7C15ull;
__host__ __device__ __forceinline__ u64 mix64(u64 z) {
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}

// ---------------------------------------------------------------------------
// warp helpers
__device__ __forceinline__ u32 lane_id() { return threadIdx.x & 31; }
__device__ __forceinline__ u32 warp_id() { return threadIdx.x >> 5; }

template <class O>
__device__ __forceinline__ u64 warp_reduce(u64 v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v = O::apply(v, __shfl_xor_sync(0xffffffffu, v, o));
  return v;
}
template <class O>
__device__ __forceinline__ u64 warp_incl_scan(u64 v) {
  const u32 lane = lane_id();
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    u64 t = __shfl_up_sync(0xffffffffu, v, o);
    if (lane >= (u32)o) v = O::apply(v, t);
  }
  return v;
}

// ---------------------------------------------------------------------------
// decoupled look-back tile status, O(#CTAs) and reusable (see scan.cu)
struct TileSlot {
  u64 agg;
  u64 incl;
  u32 flag;  // (epoch << 2) | state ; epoch = tile + 1
  u32 pad[3];
};
enum : u32 { SLOT_BUSY = 0, SLOT_AGG = 1, SLOT_INCL = 2 };

}  // namespace pip
