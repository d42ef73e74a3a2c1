// Decoupled look-back over O(#CTAs) reusable tile-status slots.
//
// Persistent kernels walk tiles round-robin (tile t on CTA t % G, wave t / G).
// Tile t publishes into slot t % R of a ring of R = 4G slots, so the scratch
// is O(#CTAs) regardless of n — the device analogue of the reference's
// O(log n) recursion stack (strong.py:107-129), never metered.  One warp
// reads 32 predecessor slots per L2 round trip.
//
// Measured (B200, scan of 2^32 words, PIP_TIMING=1 counters): the chain of
// inclusive prefixes is the kernels' serial part — ~2 look-back reads per
// tile, and under full HBM streaming one L2 round trip costs ~1.6 us; with a
// single look-back warp that also streams the tiles in, that warp was busy
// 84% of the time and set the pace (14.0 ms; 10.6 ms with the look-back
// removed, measurement only).  What helped: slots spaced `stride` apart in
// memory (14.0 -> 12.9 ms); a separate producer warp plus several look-back
// warps taking tiles round-robin, so consecutive look-backs of a CTA overlap,
// with the compute warps two tiles ahead of the stores (scan_ws2_kernel,
// filter_ws2_kernel: 12.9 -> 11.2 ms, filter 12.5 -> 10.4 ms).  What did
// not: 128-slot windows (4 loads per lane: 19 ms), block-wide windows,
// smaller tiles (more waves), 2-stage 96 KiB tiles, clusters of 2-4 CTAs
// sharing one chain step (18 ms), pairs of tiles per chain step (13.9 ms).
//
// A slot is 16 bytes {value, (epoch << 2) | state} published with ONE 128-bit
// store and read with ONE 128-bit load, so a reader always sees a value
// together with the flag it was published under (no fences, no seqlock).
// Protocol, per tile t (epoch e = t + 1):
//   writer: reuse rule — the slot last held tile u = t - R; before
//           overwriting it, wait until tile u + 1 published its inclusive
//           prefix (tile u + 1 is the only reader that cannot skip past u);
//           then store (agg, e|AGG); look back; store (incl, e|INCL).
//   reader of tile u: epoch older -> not ready; epoch newer -> overwritten
//           (restart the look-back: an overwritten slot u implies INCL(u+1)
//           exists, so restarts terminate); epoch equal -> use the value.
// All spins are bounded: a CTA that waits ~seconds sets `abort` and exits,
// so a protocol bug can never wedge the GPU.
#pragma once
#include "common.cuh"

namespace pip {

// measurement counters (PIP_TIMING=1), one copy per translation unit
static __device__ u64 g_scan_prof[8];
static __device__ u32 g_prof_on;
static __device__ u32 g_prof_cta;

struct LookbackCtx {
  TileSlot* slots;  // [R]
  u32* abort;       // global abort flag (0 = ok)
  u32 R;            // ring size (4 x resident CTAs)
  u32 stride = 1;   // slots apart in memory (spreads a look-back window over L2 lines)
};

__device__ __forceinline__ TileSlot* slot_of(const LookbackCtx& c, u64 tile) {
  return c.slots + (tile % c.R) * c.stride;
}

static constexpr bool LB_BLOCK = false;  // block-wide look-back (measured slower)
static constexpr u64 SPIN_LIMIT = 1ull << 25;  // x ~64 ns sleep => seconds

__device__ __forceinline__ bool spin_tick(const LookbackCtx& c, u64& spins) {
  if (++spins > 256) __nanosleep(32);
  if ((spins & 1023) == 0) {
    if (ld_relaxed_u32(c.abort)) return false;
    if (spins > SPIN_LIMIT) {
      atomicExch(c.abort, 1u);
      return false;
    }
  }
  return true;
}

// single thread: wait for the reuse rule before tile t may use its slot
__device__ __forceinline__ bool publish_begin(const LookbackCtx& c, u64 tile) {
  const u64 R = c.R;
  if (tile >= R) {
    const u64 v = tile - R + 1;  // tile u + 1 with u = tile - R
    const TileSlot* sv = slot_of(c, v);
    u64 spins = 0;
    for (;;) {
      u64 val, f;
      ld_slot(sv, val, f);
      const u64 e = f >> 2;
      if (e > v + 1 || (e == v + 1 && (f & 3) == SLOT_INCL)) break;
      if (!spin_tick(c, spins)) return false;
    }
  }
  return true;
}

__device__ __forceinline__ void publish_agg(const LookbackCtx& c, u64 tile, u64 agg) {
  st_slot(slot_of(c, tile), agg, ((tile + 1) << 2) | SLOT_AGG);
}

__device__ __forceinline__ void publish_incl(const LookbackCtx& c, u64 tile, u64 incl) {
  st_slot(slot_of(c, tile), incl, ((tile + 1) << 2) | SLOT_INCL);
}

enum : int { RD_NOTREADY = 0, RD_AGG = 1, RD_INCL = 2, RD_OVERWRITTEN = 3 };

template <class O>
__device__ __forceinline__ int read_slot(const LookbackCtx& c, long long u, u64& v) {
  if (u < 0) {
    v = O::identity;
    return RD_INCL;
  }
  u64 f;
  ld_slot(slot_of(c, (u64)u), v, f);
  const u64 e = f >> 2, want = (u64)u + 1;
  if (e < want) return RD_NOTREADY;
  if (e > want) return RD_OVERWRITTEN;
  const u64 st = f & 3;
  if (st == SLOT_AGG) return RD_AGG;
  if (st == SLOT_INCL) return RD_INCL;
  return RD_NOTREADY;
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
      const u32 bad = __ballot_sync(0xffffffffu, st == RD_NOTREADY);
      const u32 ow = __ballot_sync(0xffffffffu, st == RD_OVERWRITTEN);
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
    const u64 contrib = ((need >> lane) & 1u) ? v : O::identity;
    prefix = O::apply(prefix, warp_reduce<O>(contrib));
    if (incl_mask) break;
    base -= 32;
  }
  prefix_out = prefix;
  return true;
}

// whole CTA (T threads, T/32 warps): exclusive prefix of `tile`.  s_lb needs
// 3*(T/32)+2 words of shared memory.  Every thread gets the result.
template <class O, int T>
__device__ bool block_lookback(const LookbackCtx& c, u64 tile, u64& prefix_out, u64* s_lb) {
  constexpr int NW = T / 32;
  const u32 lane = lane_id(), warp = warp_id(), tid = threadIdx.x;
  u64* s_first = s_lb;               // [NW] first INCL index in warp (or 32*NW sentinel)
  u64* s_flags = s_lb + NW;          // [NW] bit0: not-ready, bit1: overwritten (positions)
  u64* s_val = s_lb + 2 * NW;        // [NW] partial folds
  u64* s_ctl = s_lb + 3 * NW;        // [2] control
  u64 prefix = O::identity;
  long long base = (long long)tile - 1;
  u64 spins = 0;
  for (;;) {
    const long long u = base - (long long)tid;
    u64 v = O::identity;
    const int st = read_slot<O>(c, u, v);
    // first INCL position (global index tid) over the block
    const u32 im = __ballot_sync(0xffffffffu, st == RD_INCL);
    if (lane == 0) s_first[warp] = im ? (u64)(warp * 32 + __ffs(im) - 1) : (u64)T;
    __syncthreads();
    u64 first = T;
#pragma unroll
    for (int w = 0; w < NW; ++w) first = s_first[w] < first ? s_first[w] : first;
    const bool in_need = (u64)tid <= first;
    const u32 bad = __ballot_sync(0xffffffffu, in_need && st == RD_NOTREADY);
    const u32 ow = __ballot_sync(0xffffffffu, in_need && st == RD_OVERWRITTEN);
    const u64 contrib = in_need ? v : O::identity;
    const u64 wsum = warp_reduce<O>(contrib);
    if (lane == 0) {
      s_flags[warp] = (bad ? 1u : 0u) | (ow ? 2u : 0u);
      s_val[warp] = wsum;
    }
    __syncthreads();
    u64 flags = 0, tot = O::identity;
#pragma unroll
    for (int w = 0; w < NW; ++w) {
      flags |= s_flags[w];
      tot = O::apply(tot, s_val[w]);
    }
    if (flags & 3) {
      // retry: a needed predecessor has not published yet (bit 0), or a
      // needed slot was recycled (bit 1: INCL(u+1) exists, start over).
      // Thread 0 decides about aborting so the whole CTA leaves together.
      if (tid == 0) s_ctl[0] = spin_tick(c, spins) ? 1 : 0;
      __syncthreads();
      const bool ok = s_ctl[0] != 0;
      __syncthreads();
      if (!ok) return false;
      if (flags & 2) {
        prefix = O::identity;
        base = (long long)tile - 1;
      }
      continue;
    }
    __syncthreads();  // s_lb reused by the next iteration
    prefix = O::apply(prefix, tot);
    if (first < (u64)T) break;
    base -= T;
  }
  prefix_out = prefix;
  return true;
}

}  // namespace pip
