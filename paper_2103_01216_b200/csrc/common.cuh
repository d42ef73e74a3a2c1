// Shared device helpers for the PIP kernels (sm_100a).
#pragma once
#include <cstdint>
#include <cuda_runtime.h>
#include "../../include/pip.h"

typedef unsigned long long u64;
typedef unsigned int u32;

namespace pip {

// random permutation progress reporting (host-buffer entry point): the
// kernel writes the highest pending id to `dev` (host-mapped; `host` is the
// same word seen from the host) after every round; rp_device calls
// hook(ctx, *host) while the rounds run
struct RpProgress {
  unsigned long long* dev;
  volatile unsigned long long* host;
  void (*hook)(void* ctx, unsigned long long top);
  void* ctx;
};


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
  u32 tz;      // MOD_EQ: trailing zeros of the divisor d = 2^tz * d_odd
  u64 inv;     // MOD_EQ: d_odd^-1 mod 2^64
  u64 lim;     // MOD_EQ: floor((2^64 - 1) / d_odd)
};
// predicate classes the filter kernels are specialised on
enum : int { PC_MASK = 0, PC_MOD = 1, PC_GEN = 2, PC_MODODD = 3, PC_MODODD0 = 4 };
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

// class-specialised predicate.  PC_MOD tests x % d == r by divisibility:
// (x - r) is a multiple of d = 2^tz * d_odd iff its low tz bits are zero and
// ((x - r) >> tz) * d_odd^-1 (mod 2^64) <= (2^64 - 1) / d_odd — one 64-bit
// multiply-low and a compare (Granlund & Montgomery).  r < d is guaranteed
// by the host (r >= d never matches and is mapped to PC_MASK false).
template <int PC>
__device__ __forceinline__ bool pred_eval_t(const DevPred& p, u64 x) {
  bool r;
  if (PC == PC_MASK) {
    r = (x & p.a) == p.b;
  } else if (PC == PC_MOD) {  // branch-free (bitwise &): no divergent short-circuit
    const u64 y = x - p.b;
    r = (x >= p.b) & ((y & ((1ull << p.tz) - 1ull)) == 0) & ((y >> p.tz) * p.inv <= p.lim);
  } else if (PC == PC_MODODD) {  // odd divisor: x = b (mod d) <=> (x - b) * d^-1 <= lim
    r = (x >= p.b) & ((x - p.b) * p.inv <= p.lim);
  } else if (PC == PC_MODODD0) {  // odd divisor, remainder 0
    r = x * p.inv <= p.lim;
  } else {
    return pred_eval(p, x);
  }
  return r != (p.negate != 0);
}

// the same test without the negate flag (callers that evaluate many words
// apply it once to the whole keep mask); PC_GEN still applies it itself
template <int PC>
__device__ __forceinline__ bool pred_raw_t(const DevPred& p, u64 x) {
  if (PC == PC_MASK) return (x & p.a) == p.b;
  if (PC == PC_MOD) {
    const u64 y = x - p.b;
    return (x >= p.b) & ((y & ((1ull << p.tz) - 1ull)) == 0) & ((y >> p.tz) * p.inv <= p.lim);
  }
  if (PC == PC_MODODD) return (x >= p.b) & ((x - p.b) * p.inv <= p.lim);
  if (PC == PC_MODODD0) return x * p.inv <= p.lim;
  return pred_eval(p, x);
}

// ---------------------------------------------------------------------------
// runtime.Rng (SplitMix64 finalizer over a golden-ratio counter)
static constexpr u64 GOLDEN = 0x9E3779B97F4A7C15ull;
__host__ __device__ __forceinline__ u64 mix64(u64 z) {
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}

__device__ __forceinline__ u64 globaltimer_ns() {
  u64 t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}
bool timing_enabled();  // env PIP_TIMING=1: per-phase timers printed to stderr
u32 lb_stride(int sms, int grid);  // look-back slot spacing in memory

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
// 16 bytes, written and read as ONE scalar .b128 access each (PTX ISA 8.3+):
// a relaxed .gpu-scope b128 load or store is a single memory operation, so it
// is single-copy atomic and value and (epoch << 2 | state) are always seen
// together.  (A .v2.u64 vector access would be two operations to the memory
// model even though it issues the same LDG/STG.E.128.STRONG.GPU.)
struct __align__(16) TileSlot {
  u64 value;
  u64 flag;  // (epoch << 2) | state ; epoch = tile + 1
};
enum : u32 { SLOT_BUSY = 0, SLOT_AGG = 1, SLOT_INCL = 2 };
__device__ __forceinline__ void st_slot(TileSlot* s, u64 value, u64 flag) {
  asm volatile(
      "{\n\t.reg .b128 t;\n\tmov.b128 t, {%1, %2};\n\t"
      "st.relaxed.gpu.global.b128 [%0], t;\n\t}" ::"l"(s),
      "l"(value), "l"(flag)
      : "memory");
}
__device__ __forceinline__ void ld_slot(const TileSlot* s, u64& value, u64& flag) {
  asm volatile(
      "{\n\t.reg .b128 t;\n\tld.relaxed.gpu.global.b128 t, [%2];\n\t"
      "mov.b128 {%0, %1}, t;\n\t}"
      : "=l"(value), "=l"(flag)
      : "l"(s)
      : "memory");
}

}  // namespace pip

// ---------------------------------------------------------------------------
// TMA bulk copies (cp.async.bulk, 1-D, no tensor map) + mbarriers (sm_90+)
namespace pip {
__device__ __forceinline__ u32 smem_u32(const void* p) {
  return (u32)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ void mbar_init(u64* bar, u32 count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}
__device__ __forceinline__ void mbar_fence_init() {
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
__device__ __forceinline__ void mbar_expect_tx(u64* bar, u32 bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)),
               "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_wait(u64* bar, u32 phase) {
  asm volatile(
      "{\n\t.reg .pred p;\n"
      "WAIT_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
      "@!p bra WAIT_%=;\n}" ::"r"(smem_u32(bar)),
      "r"(phase)
      : "memory");
}
#ifndef PIP_WAIT_NS
#define PIP_WAIT_NS 0  // 0: plain try_wait in the pipelines' wait loops
#endif
// a probe that lets the hardware suspend the thread for up to `ns`
// nanoseconds while the phase is incomplete (fewer issue slots spent on
// waiting warps; callers still see their abort flag at least every `ns`)
__device__ __forceinline__ bool mbar_try_sleep(u64* bar, u32 phase, u32 ns) {
  u32 ok;
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2, %3;\n\t"
      "selp.u32 %0, 1, 0, p;\n}"
      : "=r"(ok)
      : "r"(smem_u32(bar)), "r"(phase), "r"(ns)
      : "memory");
  return ok != 0;
}
// one non-blocking probe of the phase with parity `phase`
__device__ __forceinline__ bool mbar_try(u64* bar, u32 phase) {
  u32 ok;
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
      "selp.u32 %0, 1, 0, p;\n}"
      : "=r"(ok)
      : "r"(smem_u32(bar)), "r"(phase)
      : "memory");
  return ok != 0;
}
// global -> shared bulk copy completing on `bar` (16-byte aligned, size % 16 == 0)
__device__ __forceinline__ void tma_load_1d(void* sdst, const void* gsrc, u32 bytes, u64* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
          smem_u32(sdst)),
      "l"(gsrc), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}
// named barrier over a subset of the CTA's warps (id 1..15)
__device__ __forceinline__ void named_bar(u32 id, u32 threads) {
  asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(threads) : "memory");
}
__device__ __forceinline__ void mbar_arrive(u64* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
// 8-byte asynchronous global->shared copies (per-thread groups)
__device__ __forceinline__ void cp_async8(void* sdst, const void* gsrc) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(smem_u32(sdst)),
               "l"(gsrc)
               : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
__device__ __forceinline__ void cp_async_wait_all() { asm volatile("cp.async.wait_all;" ::: "memory"); }

// shared -> global bulk copy (bulk-group completion; 16-byte aligned, size % 16 == 0)
__device__ __forceinline__ void tma_store_1d(void* gdst, const void* ssrc, u32 bytes) {
  asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(gdst),
               "r"(smem_u32(ssrc)), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void bulk_commit() { asm volatile("cp.async.bulk.commit_group;" ::: "memory"); }
// the shared source of every committed bulk store has been read
__device__ __forceinline__ void bulk_wait_read_all() {
  asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
}
// every committed bulk store has completed
__device__ __forceinline__ void bulk_wait_all() { asm volatile("cp.async.bulk.wait_group 0;" ::: "memory"); }
// order generic-proxy accesses (all state spaces) before later async-proxy ones
__device__ __forceinline__ void fence_proxy_async_all() { asm volatile("fence.proxy.async;" ::: "memory"); }
// order prior generic-proxy shared-memory accesses before async-proxy (TMA) ones
__device__ __forceinline__ void fence_proxy_async_smem() {
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}
__device__ __forceinline__ ulonglong2 lds2(const u64* p) {
  return *reinterpret_cast<const ulonglong2*>(p);
}
}  // namespace pip
