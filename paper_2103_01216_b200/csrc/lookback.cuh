// Decoupled look-back over O(#CTAs) reusable tile-status slots.
//
// Persistent kernels assign tiles round-robin: tile t is processed by CTA
// t % G in wave t / G.  Each CTA owns two status slots (wave parity), so the
// scratch is 2*G slots regardless of n — the device analogue of the
// reference's O(log n) recursion stack (strong.py:107-129), never metered.
//
// Protocol (one writer per slot, many readers):
//   writer, per tile t (epoch e = t + 1):
//     0. reuse rule: the slot last held tile u = t - 2G; before overwriting
//        it wait until tile u + 1 has published its inclusive prefix (then
//        tile u + 1 — the only reader that cannot skip past u — is done
//        with it);
//     1. flag = (e, BUSY); fence; agg; fence; flag = (e, AGG)  [release]
//     2. look back; fence; incl; fence; flag = (e, INCL)        [release]
//   reader of tile u: acquire flag; epoch older -> not ready; epoch newer ->
//     overwritten (restart the look-back: an overwritten slot u implies
//     INCL(u+1) exists, so the restart terminates); epoch equal -> read the
//     value, fence, re-read the flag (seqlock) and accept iff the epoch held.
// All spins are bounded: a CTA that waits ~seconds sets `abort` and exits,
// so a protocol bug can never wedge the GPU.
#pragma once
#include "common.cuh"

namespace pip {

struct LookbackCtx {
  TileSlot* slots;  // [2 * G]
  u32* abort;       // global abort flag (0 = ok)
  u32 G;
};

__device__ __forceinline__ TileSlot* slot_of(const LookbackCtx& c, u64 tile) {
  return c.slots + ((tile % c.G) * 2 + ((tile / c.G) & 1));
}

static constexpr u64 SPIN_LIMIT = 1ull << 25;  // x ~64..256 ns sleep => seconds

__device__ __forceinline__ bool spin_tick(const LookbackCtx& c, u64& spins) {
  if (++spins > 64) __nanosleep(64);
  if ((spins & 1023) == 0) {
    if (ld_relaxed_u32(c.abort)) return false;
    if (spins > SPIN_LIMIT) {
      atomicExch(c.abort, 1u);
      return false;
    }
  }
  return true;
}

// single thread: wait for the reuse rule, then mark the slot busy for tile t
__device__ __forceinline__ bool publish_begin(const LookbackCtx& c, u64 tile) {
  TileSlot* s = slot_of(c, tile);
  const u64 G = c.G;
  if (tile >= 2 * G) {
    const u64 v = tile - 2 * G + 1;  // tile u + 1 with u = tile - 2G
    TileSlot* sv = slot_of(c, v);
    u64 spins = 0;
    for (;;) {
      u32 f = ld_acquire_u32(&sv->flag);
      u64 e = f >> 2;
      if (e > v + 1 || (e == v + 1 && (f & 3) == SLOT_INCL)) break;
      if (!spin_tick(c, spins)) return false;
    }
  }
  st_relaxed_u32(&s->flag, (u32)((tile + 1) << 2) | SLOT_BUSY);
  fence_gpu();
  return true;
}

__device__ __forceinline__ void publish_agg(const LookbackCtx& c, u64 tile, u64 agg) {
  TileSlot* s = slot_of(c, tile);
  st_relaxed_u64(&s->agg, agg);
  fence_gpu();
  st_release_u32(&s->flag, (u32)((tile + 1) << 2) | SLOT_AGG);
}

__device__ __forceinline__ void publish_incl(const LookbackCtx& c, u64 tile, u64 incl) {
  TileSlot* s = slot_of(c, tile);
  fence_gpu();
  st_relaxed_u64(&s->incl, incl);
  fence_gpu();
  st_release_u32(&s->flag, (u32)((tile + 1) << 2) | SLOT_INCL);
}

enum : int { RD_NOTREADY = 0, RD_AGG = 1, RD_INCL = 2, RD_OVERWRITTEN = 3 };

template <class O>
__device__ __forceinline__ int read_slot(const LookbackCtx& c, long long u, u64& v) {
  if (u < 0) {
    v = O::identity;
    return RD_INCL;
  }
  TileSlot* s = slot_of(c, (u64)u);
  u32 f1 = ld_acquire_u32(&s->flag);
  u64 e = f1 >> 2, want = (u64)u + 1;
  if (e < want) return RD_NOTREADY;
  if (e > want) return RD_OVERWRITTEN;
  u32 st = f1 & 3;
  if (st == SLOT_BUSY) return RD_NOTREADY;
  v = (st == SLOT_AGG) ? ld_relaxed_u64(&s->agg) : ld_relaxed_u64(&s->incl);
  fence_gpu();
  u32 f2 = ld_relaxed_u32(&s->flag);
  if ((f2 >> 2) != e) return RD_OVERWRITTEN;
  return st == SLOT_AGG ? RD_AGG : RD_INCL;
}

// whole warp: exclusive prefix (fold of all tiles < tile); false on abort
template <class O>
__device__ bool lookback(const LookbackCtx& c, u64 tile, u64& prefix_out) {
  const u32 lane = lane_id();
  u64 prefix = O::identity;
  long long base = (long long)tile - 1;
  u64 spins = 0;
  for (;;) {
    const long long u = base - (long long)lane;
    u64 v = O::identity;
    int st;
    u32 incl_mask, need;
    bool restart = false;
    for (;;) {
      st = read_slot<O>(c, u, v);
      incl_mask = __ballot_sync(0xffffffffu, st == RD_INCL);
      u32 bad = __ballot_sync(0xffffffffu, st == RD_NOTREADY);
      u32 ow = __ballot_sync(0xffffffffu, st == RD_OVERWRITTEN);
      need = incl_mask ? (((incl_mask & (0u - incl_mask)) << 1) - 1u) : 0xffffffffu;
      if (ow & need) {
        restart = true;
        break;
      }
      if ((bad & need) == 0) break;
      bool ok = true;
      if (lane == 0) ok = spin_tick(c, spins);
      if (!__shfl_sync(0xffffffffu, (int)ok, 0)) return false;
    }
    if (restart) {
      prefix = O::identity;
      base = (long long)tile - 1;
      bool ok = true;
      if (lane == 0) ok = spin_tick(c, spins);
      if (!__shfl_sync(0xffffffffu, (int)ok, 0)) return false;
      continue;
    }
    u64 contrib = ((need >> lane) & 1u) ? v : O::identity;
    prefix = O::apply(prefix, warp_reduce<O>(contrib));
    if (incl_mask) break;
    base -= 32;
  }
  prefix_out = prefix;
  return true;
}

}  // namespace pip
