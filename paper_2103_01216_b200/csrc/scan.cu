// In-place scan / reduce (strong.scan, strong.scan_blocked, strong.reduce).
//
// Reference: pkg/src/pipal/strong.py:101-166 (Alg. 3 up/down sweep kept
// inside the array) and :169-236 (blocked variant).  Both compute the
// exclusive scan mod 2^64 plus the total; this file computes the same
// result in ONE pass over HBM (read 8 B + write 8 B per element): a
// persistent grid walks 8192-element tiles round-robin, reduces each tile,
// publishes its aggregate, resolves its prefix by decoupled look-back over
// O(#CTAs) status slots (lookback.cuh), then scans the tile with warp
// shuffles and writes it back in place.
//
// Layout per tile (512 threads = 16 warps): warp w owns the contiguous
// segment [tile*8192 + w*512, +512); in chunk j (0..7) lane l holds the pair
// (2l, 2l+1) of the 64-element sub-chunk j, loaded/stored as one 128-bit
// access, so every warp access is a fully coalesced 512-byte transaction.
#include <cstdio>
#include <cstdlib>
#include "lookback.cuh"

namespace pip {

static constexpr int SCAN_THREADS = 512;
static constexpr int SCAN_ITEMS = 16;
static constexpr u64 SCAN_TILE = (u64)SCAN_THREADS * SCAN_ITEMS;  // 8192

// One tile, values already in registers (x[2j], x[2j+1] = pair j of this
// lane in its warp's 512-element segment).  Publishes the aggregate, looks
// back, scans with warp shuffles and stores.  false => abort.
template <int OP, bool INCLUSIVE, int THREADS>
__device__ __forceinline__ bool scan_tile_body(const u64 (&x)[SCAN_ITEMS], u64* __restrict__ a,
                                               u64 n, u64 tile, u64 init, const u64* carry_in,
                                               u64* total, const LookbackCtx& c, u64 num_tiles,
                                               bool full, u64* s_warp, int* s_abort) {
  using O = Op<OP>;
  constexpr u64 TILE = (u64)THREADS * SCAN_ITEMS;
  constexpr int NW = THREADS / 32;
  const u32 lane = lane_id(), warp = warp_id();
  const u64 wbase = tile * TILE + (u64)warp * 512;
  u64* s_ctl = s_warp + NW;      // [2]: agg, ok
  u64* s_lb = s_warp + NW + 2;   // block look-back scratch
  u64 t = x[0];
#pragma unroll
  for (int k = 1; k < SCAN_ITEMS; ++k) t = O::apply(t, x[k]);
  t = warp_reduce<O>(t);
  if (lane == 0) s_warp[warp] = t;
  __syncthreads();
  // carry_in (streaming chunks, shards) acts as an inclusive tile -1
  u64 prefix = (tile == 0 && carry_in) ? *carry_in : O::identity;
  if (warp == 0) {
    const u64 wv = lane < NW ? s_warp[lane] : O::identity;
    const u64 winc = warp_incl_scan<O>(wv);
    u64 wexc = __shfl_up_sync(0xffffffffu, winc, 1);
    if (lane == 0) wexc = O::identity;
    const u64 agg = __shfl_sync(0xffffffffu, winc, NW - 1);
    __syncwarp();
    if (lane < NW) s_warp[lane] = wexc;
    if (lane == 0) {
      const int ok = publish_begin(c, tile);
      if (ok) {
        if (tile == 0) publish_incl(c, tile, O::apply(prefix, agg));
        else publish_agg(c, tile, agg);
      }
      s_ctl[0] = agg;
      s_ctl[1] = ok;
    }
  }
  __syncthreads();
  const u64 agg = s_ctl[0];
  bool ok = s_ctl[1] != 0;
  if (ok && tile > 0) {
    if (LB_BLOCK) {
      ok = block_lookback<O, THREADS>(c, tile, prefix, s_lb);
    } else {
      // warp 0 looks back; the prefix reaches the CTA through shared memory
      if (warp == 0) {
        const bool wok = lookback<O>(c, tile, prefix);
        if (lane == 0) {
          s_lb[0] = prefix;
          s_lb[1] = wok;
        }
      }
      __syncthreads();
      prefix = s_lb[0];
      ok = s_lb[1] != 0;
    }
    if (ok && threadIdx.x == 0) publish_incl(c, tile, O::apply(prefix, agg));
  }
  if (!ok) {
    if (threadIdx.x == 0) atomicExch(c.abort, 1u);
    return false;
  }
  if (threadIdx.x == 0 && tile == num_tiles - 1 && total) *total = O::apply(prefix, agg);
  (void)s_abort;
  u64 run = O::apply(prefix, s_warp[warp]);
#pragma unroll
  for (int j = 0; j < 8; ++j) {
    const u64 x0 = x[2 * j], x1 = x[2 * j + 1];
    const u64 s = O::apply(x0, x1);
    const u64 inc = warp_incl_scan<O>(s);
    u64 exc = __shfl_up_sync(0xffffffffu, inc, 1);
    if (lane == 0) exc = O::identity;
    const u64 tot = __shfl_sync(0xffffffffu, inc, 31);
    const u64 e = O::apply(run, exc);
    u64 o0, o1;
    if (INCLUSIVE) {
      o0 = O::apply(e, x0);
      o1 = O::apply(o0, x1);
    } else {
      o0 = e;
      o1 = O::apply(e, x0);
    }
    o0 = O::apply(init, o0);
    o1 = O::apply(init, o1);
    const u64 i0 = wbase + 64 * j + 2 * lane;
    if (full) {
      stg_stream2(a + i0, o0, o1);
    } else {
      if (i0 < n) a[i0] = o0;
      if (i0 + 1 < n) a[i0 + 1] = o1;
    }
    run = O::apply(run, tot);
  }
  __syncthreads();  // s_warp is rewritten by the next tile
  return true;
}

// register path: any alignment (VEC = 16-byte aligned base); tiles
// round-robin over the persistent grid (tile t on CTA t % G)
template <int OP, bool INCLUSIVE, bool VEC>
__global__ void __launch_bounds__(SCAN_THREADS, 2)
scan_kernel(u64* __restrict__ a, u64 n, u64 init, const u64* carry_in, u64* total, LookbackCtx c,
            u64 num_tiles, u32* counter) {
  using O = Op<OP>;
  __shared__ u64 s_warp[4 * (SCAN_THREADS / 32) + 4];
  __shared__ int s_abort;
  const u32 lane = lane_id(), warp = warp_id();
  (void)counter;
  for (u64 tile = blockIdx.x; tile < num_tiles; tile += gridDim.x) {
    const u64 wbase = tile * SCAN_TILE + (u64)warp * 512;
    const bool full = VEC && (tile * SCAN_TILE + SCAN_TILE <= n);
    u64 x[SCAN_ITEMS];
    if (full) {
#pragma unroll
      for (int j = 0; j < 8; ++j) {
        ulonglong2 v = ldg_stream2(a + wbase + 64 * j + 2 * lane);
        x[2 * j] = v.x;
        x[2 * j + 1] = v.y;
      }
    } else {
#pragma unroll
      for (int j = 0; j < 8; ++j) {
        const u64 i0 = wbase + 64 * j + 2 * lane;
        x[2 * j] = i0 < n ? a[i0] : O::identity;
        x[2 * j + 1] = i0 + 1 < n ? a[i0 + 1] : O::identity;
      }
    }
    if (!scan_tile_body<OP, INCLUSIVE, SCAN_THREADS>(x, a, n, tile, init, carry_in, total, c,
                                                     num_tiles, full, s_warp, &s_abort))
      return;
  }
}

// TMA path (16-byte aligned base): each CTA keeps STAGES claimed tiles in
// flight as cp.async.bulk copies into a shared-memory ring, so HBM reads
// overlap the look-back and scan of the current tile.
template <int OP, bool INCLUSIVE, int THREADS, int STAGES>
__global__ void __launch_bounds__(THREADS, 1)
scan_tma_kernel(u64* __restrict__ a, u64 n, u64 init, const u64* carry_in, u64* total,
                LookbackCtx c, u64 num_tiles, u64 full_tiles, u32* counter) {
  using O = Op<OP>;
  constexpr u64 TILE = (u64)THREADS * SCAN_ITEMS;
  constexpr u32 TILE_BYTES = (u32)(TILE * 8);
  extern __shared__ __align__(128) u64 ring[];
  __shared__ __align__(8) u64 bars[STAGES];
  __shared__ u64 s_tile[STAGES];
  __shared__ u64 s_warp[4 * (THREADS / 32) + 4];
  __shared__ int s_abort;
  const u32 tid = threadIdx.x, lane = lane_id(), warp = warp_id();
  if (tid == 0) {
    for (int s = 0; s < STAGES; ++s) mbar_init(&bars[s], 1);
    mbar_fence_init();
  }
  __syncthreads();
  auto issue = [&](u64 k) {  // tid 0: start the copy of this CTA's k-th tile
    const int s = (int)(k % STAGES);
    const u64 t = blockIdx.x + k * gridDim.x;
    s_tile[s] = t;
    if (t < full_tiles) {
      mbar_expect_tx(&bars[s], TILE_BYTES);
#pragma unroll
      for (int q = 0; q < 4; ++q)
        tma_load_1d(ring + s * TILE + q * (TILE / 4), a + t * TILE + q * (TILE / 4), TILE_BYTES / 4,
                    &bars[s]);
    } else {
      mbar_arrive(&bars[s]);
    }
  };
  if (tid == 0)
    for (int k = 0; k < STAGES; ++k) issue(k);
  for (u64 k = 0;; ++k) {
    const int s = (int)(k % STAGES);
    mbar_wait(&bars[s], (u32)((k / STAGES) & 1));
    const u64 tile = s_tile[s];
    if (tile >= num_tiles) break;
    u64 x[SCAN_ITEMS];
    const bool full = tile < full_tiles;
    if (full) {
      const u64* src = ring + s * TILE + warp * 512;
#pragma unroll
      for (int j = 0; j < 8; ++j) {
        const ulonglong2 v = lds2(src + 64 * j + 2 * lane);
        x[2 * j] = v.x;
        x[2 * j + 1] = v.y;
      }
    } else {
      const u64 wbase = tile * TILE + (u64)warp * 512;
#pragma unroll
      for (int j = 0; j < 8; ++j) {
        const u64 i0 = wbase + 64 * j + 2 * lane;
        x[2 * j] = i0 < n ? a[i0] : O::identity;
        x[2 * j + 1] = i0 + 1 < n ? a[i0 + 1] : O::identity;
      }
    }
    __syncthreads();  // stage s is in registers: refill it
    if (tid == 0) {
      fence_proxy_async_smem();
      issue(k + STAGES);
    }
    if (!scan_tile_body<OP, INCLUSIVE, THREADS>(x, a, n, tile, init, carry_in, total, c, num_tiles,
                                                full, s_warp, &s_abort))
      return;
  }
}

// Aggregate-ahead pipeline (16-byte aligned base, whole tiles only):
// every CTA keeps STAGES of its tiles in flight as cp.async.bulk copies into
// a shared-memory ring and, before it looks back for tile k, reduces tile
// k+1 (already in shared memory) and publishes that aggregate.  So when any
// tile looks back, the tiles of its wave published their aggregates one
// iteration earlier: the look-back never waits for a predecessor's HBM load,
// only for L2 round trips.  (The measured bottleneck of the plain kernel was
// exactly that wait: 51% of warp stalls at the CTA barrier behind warp 0's
// look-back, profiles/r01_scan_v1_lookback_stall.ncu-rep.)
template <int OP, bool INCLUSIVE, int THREADS, int STAGES>
__global__ void __launch_bounds__(THREADS, 1)
scan_ahead_kernel(u64* __restrict__ a, u64 init, const u64* carry_in, u64* total, LookbackCtx c,
                  u64 num_tiles) {
  using O = Op<OP>;
  constexpr int NW = THREADS / 32;
  constexpr u64 TILE = (u64)THREADS * SCAN_ITEMS;
  constexpr u32 TILE_BYTES = (u32)(TILE * 8);
  static_assert(STAGES >= 2, "need a stage for the tile ahead");
  extern __shared__ __align__(128) u64 ring[];
  __shared__ __align__(8) u64 bars[STAGES];
  __shared__ u64 s_wexc[STAGES][NW];
  __shared__ u64 s_agg[STAGES];
  __shared__ u64 s_tmp[NW + 4];
  const u32 tid = threadIdx.x, lane = lane_id(), warp = warp_id();
  const u64 G = gridDim.x;
  if (tid == 0) {
    for (int s = 0; s < STAGES; ++s) mbar_init(&bars[s], 1);
    mbar_fence_init();
  }
  __syncthreads();
  auto issue = [&](u64 k) {
    const u64 t = blockIdx.x + k * G;
    if (t < num_tiles) {
      const int s = (int)(k % STAGES);
      mbar_expect_tx(&bars[s], TILE_BYTES);
#pragma unroll
      for (int q = 0; q < 4; ++q)
        tma_load_1d(ring + s * TILE + q * (TILE / 4), a + t * TILE + q * (TILE / 4), TILE_BYTES / 4,
                    &bars[s]);
    }
  };
  // wait for the k-th tile, fold it: s_agg[stage], s_wexc[stage][warp]
  auto reduce_stage = [&](u64 k) {
    const int s = (int)(k % STAGES);
    mbar_wait(&bars[s], (u32)((k / STAGES) & 1));
    const u64* src = ring + s * TILE + warp * 512;
    u64 t = O::identity;
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      const ulonglong2 v = lds2(src + 64 * j + 2 * lane);
      t = O::apply(t, O::apply(v.x, v.y));
    }
    t = warp_reduce<O>(t);
    if (lane == 0) s_tmp[warp] = t;
    __syncthreads();
    if (warp == 0) {
      const u64 wv = lane < NW ? s_tmp[lane] : O::identity;
      const u64 winc = warp_incl_scan<O>(wv);
      u64 wexc = __shfl_up_sync(0xffffffffu, winc, 1);
      if (lane == 0) wexc = O::identity;
      if (lane < NW) s_wexc[s][lane] = wexc;
      if (lane == NW - 1) s_agg[s] = winc;
    }
    __syncthreads();
  };
  if (tid == 0)
    for (int k = 0; k < STAGES; ++k) issue(k);
  if ((u64)blockIdx.x >= num_tiles) return;
  // first tile: publish its aggregate (tile 0: its inclusive prefix)
  reduce_stage(0);
  if (tid == 0) {
    const u64 t0 = blockIdx.x;
    const int ok = publish_begin(c, t0);
    if (ok) {
      if (t0 == 0) publish_incl(c, 0, O::apply(carry_in ? *carry_in : O::identity, s_agg[0]));
      else publish_agg(c, t0, s_agg[0]);
    }
    s_tmp[NW] = ok;
  }
  __syncthreads();
  if (!s_tmp[NW]) return;
  for (u64 k = 0;; ++k) {
    const u64 tile = blockIdx.x + k * G;
    if (tile >= num_tiles) break;
    const int s = (int)(k % STAGES);
    const u64 tn = tile + G;
    // (1) the next tile's aggregate goes out before we wait on anyone
    if (tn < num_tiles) {
      reduce_stage(k + 1);
      if (tid == 0) {
        const int ok = publish_begin(c, tn);
        if (ok) publish_agg(c, tn, s_agg[(k + 1) % STAGES]);
        s_tmp[NW] = ok;
      }
    }
    // (2) this tile's prefix
    if (warp == 0) {
      u64 prefix = (tile == 0 && carry_in) ? *carry_in : O::identity;
      bool ok = true;
      if (tile > 0) {
        ok = lookback<O>(c, tile, prefix);
        if (ok && lane == 0) publish_incl(c, tile, O::apply(prefix, s_agg[s]));
      }
      if (lane == 0) {
        s_tmp[NW + 1] = prefix;
        s_tmp[NW + 2] = ok;
        if (ok && tile == num_tiles - 1 && total) *total = O::apply(prefix, s_agg[s]);
      }
    }
    __syncthreads();
    if (!s_tmp[NW + 2] || (tn < num_tiles && !s_tmp[NW])) {
      if (tid == 0) atomicExch(c.abort, 1u);
      return;
    }
    // (3) scan the tile out of shared memory and store it
    u64 run = O::apply(s_tmp[NW + 1], s_wexc[s][warp]);
    const u64* src = ring + s * TILE + warp * 512;
    const u64 wbase = tile * TILE + (u64)warp * 512;
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      const ulonglong2 v = lds2(src + 64 * j + 2 * lane);
      const u64 x0 = v.x, x1 = v.y;
      const u64 inc = warp_incl_scan<O>(O::apply(x0, x1));
      u64 exc = __shfl_up_sync(0xffffffffu, inc, 1);
      if (lane == 0) exc = O::identity;
      const u64 tot = __shfl_sync(0xffffffffu, inc, 31);
      const u64 e = O::apply(run, exc);
      u64 o0, o1;
      if (INCLUSIVE) {
        o0 = O::apply(e, x0);
        o1 = O::apply(o0, x1);
      } else {
        o0 = e;
        o1 = O::apply(e, x0);
      }
      stg_stream2(a + wbase + 64 * j + 2 * lane, O::apply(init, o0), O::apply(init, o1));
      run = O::apply(run, tot);
    }
    // (4) release the stage
    __syncthreads();
    if (tid == 0) {
      fence_proxy_async_smem();
      issue(k + STAGES);
    }
  }
}

// Warp-specialized pipeline (16-byte aligned base, whole tiles only).
// Warp 0 is the producer / look-back warp: it keeps S-1 tiles ahead in flight
// as cp.async.bulk copies, and for tile k publishes the aggregate, looks back
// and publishes the inclusive prefix; the NWC compute warps meanwhile reduce
// tile k and scan + store tile k-1.  The look-back's L2 round trips (the
// barrier stall of every single-role kernel above, profiles/
// r01_scan_ahead_summary.txt) leave the compute warps' critical path.
// Hand-offs are mbarriers: full (TMA bytes landed), reduced (tile aggregate
// in smem), pready (prefix in smem), empty (stage stored, may be refilled).

template <int OP, bool INCLUSIVE, int NWC, int S, bool DYN, bool AHEAD = false, int WPW = 512>
__global__ void __launch_bounds__(32 * (NWC + 1), 1)
scan_ws_kernel(u64* __restrict__ a, u64 init, const u64* carry_in, u64* total, LookbackCtx c,
               u64 num_tiles, u32* counter) {
  using O = Op<OP>;
  constexpr u64 TILE = (u64)NWC * WPW;  // WPW words per compute warp
  constexpr int JW = WPW / 64;
  constexpr u32 TILE_BYTES = (u32)(TILE * 8);
  extern __shared__ __align__(128) u64 ring[];
  __shared__ __align__(8) u64 full[S], reduced[S], pready[S], empty[S];
  __shared__ u64 s_wtot[S][NWC];
  __shared__ u64 s_wexc[S][NWC];
  __shared__ u64 s_agg[S];
  __shared__ u64 s_prefix[S];
  __shared__ int s_abort;
  __shared__ u64 s_tile[S];  // DYN: tile id of each stage (claimed at issue)
  const u32 tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const u64 G = gridDim.x, B = blockIdx.x;
  if (tid == 0) {
    for (int s = 0; s < S; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&reduced[s], 1);
      mbar_init(&pready[s], 1);
      mbar_init(&empty[s], 1);
    }
    s_abort = 0;
    mbar_fence_init();
  }
  __syncthreads();
  auto issue = [&](u64 k) {  // one thread: TMA tile k into stage k % S
    const int s = (int)(k % S);
    const u64 t = DYN ? (u64)atomicAdd(counter, 1u) : B + k * G;
    s_tile[s] = t;
    if (DYN && t >= num_tiles) {
      mbar_arrive(&full[s]);
      return;
    }
    mbar_expect_tx(&full[s], TILE_BYTES);
#pragma unroll
    for (int q = 0; q < 4; ++q)
      tma_load_1d(ring + s * TILE + q * (TILE / 4), a + t * TILE + q * (TILE / 4), TILE_BYTES / 4,
                  &full[s]);
  };

  if (warp == 0) {
    // ------------------------------------------------ producer / look-back
    if (lane == 0)
      for (u64 k = 0; k + 1 < (u64)S; ++k)
        if (DYN || B + k * G < num_tiles) issue(k);
    __syncwarp();
    for (u64 k = 0;; ++k) {
      const int s = (int)(k % S);
      if (DYN) mbar_wait(&full[s], (u32)((k / S) & 1));  // s_tile[s] is set
      const u64 t = DYN ? s_tile[s] : B + k * G;
      if (t >= num_tiles) break;
      if (AHEAD) {
        // the aggregate of tile k+1 goes out before tile k looks back
        const u64 kn = k + 1, tn = DYN ? 0 : B + kn * G;
        int okn = 1;
        if (tn < num_tiles) {
          const int sn = (int)(kn % S);
          mbar_wait(&reduced[sn], (u32)((kn / S) & 1));
          if (lane == 0) {
            okn = publish_begin(c, tn);
            if (okn) publish_agg(c, tn, s_agg[sn]);
          }
          okn = __shfl_sync(0xffffffffu, okn, 0);
        }
        if (!okn) {
          if (lane == 0) {
            s_abort = 1;
            mbar_arrive(&pready[s]);
          }
          return;
        }
      }
      const u64 tw0 = clock64();
      mbar_wait(&reduced[s], (u32)((k / S) & 1));
      const u64 tw1 = clock64();
      const u64 agg = s_agg[s];
      u64 prefix = (t == 0 && carry_in) ? *carry_in : O::identity;
      int ok = 1;
      if (lane == 0 && (!AHEAD || k == 0)) {
        ok = publish_begin(c, t);
        if (ok) {
          if (t == 0) publish_incl(c, 0, O::apply(prefix, agg));
          else publish_agg(c, t, agg);
        }
      }
      ok = __shfl_sync(0xffffffffu, ok, 0);
      if (ok && t > 0) {
        ok = lookback<O>(c, t, prefix);
        if (ok && lane == 0) publish_incl(c, t, O::apply(prefix, agg));
      }
      if (lane == 0) {
        s_prefix[s] = prefix;
        if (!ok) s_abort = 1;
        if (ok && t == num_tiles - 1 && total) *total = O::apply(prefix, agg);
        mbar_arrive(&pready[s]);
        if (B == g_prof_cta && g_prof_on) {
          g_scan_prof[0] += tw1 - tw0;            // producer waits for the reduce
          g_scan_prof[1] += clock64() - tw1;      // publish + look-back
          g_scan_prof[2] += 1;
        }
      }
      if (!ok) return;
      // refill: tile k+S-1 goes into the stage of tile k-1 once that is stored
      const u64 kk = k + S - 1;
      if (DYN || B + kk * G < num_tiles) {
        if (kk >= (u64)S) mbar_wait(&empty[kk % S], (u32)(((kk / S) - 1) & 1));
        if (lane == 0) {
          fence_proxy_async_smem();
          issue(kk);
        }
      }
      __syncwarp();
    }
    return;
  }

  // ---------------------------------------------------- compute warps
  const u32 w = warp - 1;
  auto scan_store = [&](u64 k) -> bool {
    const int s = (int)(k % S);
    const u64 tp0 = clock64();
    mbar_wait(&pready[s], (u32)((k / S) & 1));
    if (B == g_prof_cta && tid == 32 && g_prof_on) g_scan_prof[3] += clock64() - tp0;  // compute waits for prefix
    if (s_abort) return false;
    u64 run = O::apply(s_prefix[s], s_wexc[s][w]);
    const u64* src = ring + s * TILE + w * WPW;
    const u64 wbase = (DYN ? s_tile[s] : B + k * G) * TILE + (u64)w * WPW;
#pragma unroll
    for (int j = 0; j < JW; ++j) {
      const ulonglong2 v = lds2(src + 64 * j + 2 * lane);
      const u64 x0 = v.x, x1 = v.y;
      const u64 inc = warp_incl_scan<O>(O::apply(x0, x1));
      u64 exc = __shfl_up_sync(0xffffffffu, inc, 1);
      if (lane == 0) exc = O::identity;
      const u64 tot = __shfl_sync(0xffffffffu, inc, 31);
      const u64 e = O::apply(run, exc);
      u64 o0, o1;
      if (INCLUSIVE) {
        o0 = O::apply(e, x0);
        o1 = O::apply(o0, x1);
      } else {
        o0 = e;
        o1 = O::apply(e, x0);
      }
      stg_stream2(a + wbase + 64 * j + 2 * lane, O::apply(init, o0), O::apply(init, o1));
      run = O::apply(run, tot);
    }
    named_bar(1, NWC * 32);  // every compute warp has read stage s
    if (w == 0 && lane == 0) mbar_arrive(&empty[s]);
    return true;
  };
  auto reduce_tile = [&](u64 k) {
    const int s = (int)(k % S);
    mbar_wait(&full[s], (u32)((k / S) & 1));
    const u64* src = ring + s * TILE + w * WPW;
    u64 acc = O::identity;
#pragma unroll
    for (int j = 0; j < JW; ++j) {
      const ulonglong2 v = lds2(src + 64 * j + 2 * lane);
      acc = O::apply(acc, O::apply(v.x, v.y));
    }
    acc = warp_reduce<O>(acc);
    if (lane == 0) s_wtot[s][w] = acc;
    named_bar(1, NWC * 32);
    if (w == 0) {
      const u64 wv = lane < (u32)NWC ? s_wtot[s][lane] : O::identity;
      const u64 winc = warp_incl_scan<O>(wv);
      u64 wexc = __shfl_up_sync(0xffffffffu, winc, 1);
      if (lane == 0) wexc = O::identity;
      if (lane < (u32)NWC) s_wexc[s][lane] = wexc;
      if (lane == NWC - 1) s_agg[s] = winc;
      __syncwarp();
      if (lane == 0) mbar_arrive(&reduced[s]);
    }
  };
  if (AHEAD && !DYN) {
    // compute warps run two tiles ahead in reducing: reduce(k+2) after store(k)
    if (B < num_tiles) reduce_tile(0);
    if (B + G < num_tiles) reduce_tile(1);
    for (u64 k = 0; B + k * G < num_tiles; ++k) {
      if (!scan_store(k)) return;
      if (B + (k + 2) * G < num_tiles) reduce_tile(k + 2);
    }
    return;
  }
  for (u64 k = 0;; ++k) {
    const int s = (int)(k % S);
    if (DYN) mbar_wait(&full[s], (u32)((k / S) & 1));
    const u64 t = DYN ? s_tile[s] : B + k * G;
    if (t >= num_tiles) {
      if (k > 0) scan_store(k - 1);
      break;
    }
    const u64 tf0 = clock64();
    if (!DYN) mbar_wait(&full[s], (u32)((k / S) & 1));
    if (B == g_prof_cta && tid == 32 && g_prof_on) g_scan_prof[4] += clock64() - tf0;  // compute waits for data
    const u64* src = ring + s * TILE + w * WPW;
    u64 acc = O::identity;
#pragma unroll
    for (int j = 0; j < JW; ++j) {
      const ulonglong2 v = lds2(src + 64 * j + 2 * lane);
      acc = O::apply(acc, O::apply(v.x, v.y));
    }
    acc = warp_reduce<O>(acc);
    if (lane == 0) s_wtot[s][w] = acc;
    named_bar(1, NWC * 32);
    if (w == 0) {
      const u64 wv = lane < (u32)NWC ? s_wtot[s][lane] : O::identity;
      const u64 winc = warp_incl_scan<O>(wv);
      u64 wexc = __shfl_up_sync(0xffffffffu, winc, 1);
      if (lane == 0) wexc = O::identity;
      if (lane < (u32)NWC) s_wexc[s][lane] = wexc;
      if (lane == NWC - 1) s_agg[s] = winc;
      __syncwarp();
      if (lane == 0) mbar_arrive(&reduced[s]);
    }
    if (k > 0 && !scan_store(k - 1)) return;
  }
}

// ---------------------------------------------------------------------------
// Same pipeline with the roles split across more warps: warp 0 only streams
// tiles in, LBW look-back warps take tiles round-robin (warp 1 + (k % LBW)),
// so the look-backs of consecutive tiles of this CTA overlap instead of
// queueing behind one another (the single look-back warp of scan_ws_kernel
// is busy ~84% of the time at 2^32).
// TK: tiles are handed out by ticket (one atomic per tile, drawn by the
// producer one tile ahead) instead of round-robin B + k G: a CTA on a slower
// SM then takes fewer tiles instead of holding every look-back chain up.
template <int OP, bool INCLUSIVE, int NWC, int S, int LBW, int D = 1, int MB = 1, bool TK = false>
__global__ void __launch_bounds__(32 * (NWC + 1 + LBW), MB)
scan_ws2_kernel(u64* __restrict__ a, u64 init, const u64* carry_in, u64* total, LookbackCtx c,
                u64 num_tiles, u32* ticket) {
  using O = Op<OP>;
  constexpr u64 TILE = (u64)NWC * 512;
  constexpr u32 TILE_BYTES = (u32)(TILE * 8);
  extern __shared__ __align__(128) u64 ring[];
  __shared__ __align__(8) u64 full[S], reduced[S], pready[S], empty[S];
  __shared__ u64 s_wtot[S][NWC];
  __shared__ u64 s_wexc[S][NWC];
  __shared__ u64 s_agg[S];
  __shared__ u64 s_prefix[S];
  __shared__ volatile int s_abort;
  __shared__ volatile u64 s_tile[S];  // TK: the tile in each stage (>= num_tiles: the stream's end)
  __shared__ volatile int s_done;     // TK: every tile of this CTA is stored; look-back warps leave
  const u32 tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const u64 G = gridDim.x, B = blockIdx.x;
  if (tid == 0) {
    for (int s = 0; s < S; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&reduced[s], 1);
      mbar_init(&pready[s], 1);
      mbar_init(&empty[s], 1);
    }
    s_abort = 0;
    s_done = 0;
    mbar_fence_init();
  }
  __syncthreads();
  auto ph = [&](u64 k) { return (u32)((k / S) & 1); };
  auto wait_or_abort = [&](u64* bar, u32 phase) -> bool {
    while (!(PIP_WAIT_NS ? mbar_try_sleep(bar, phase, PIP_WAIT_NS) : mbar_try(bar, phase)))
      if (s_abort || (TK && s_done)) return false;
    return true;
  };
  auto tile_of = [&](u64 k) -> u64 { return TK ? s_tile[k % S] : B + k * G; };
  if (warp == 0) {
    // ------------------------------------------------------------ producer
    u64 tnext = 0;
    if (TK && lane == 0) tnext = atomicAdd(ticket, 1u);
    for (u64 k = 0; TK || B + k * G < num_tiles; ++k) {
      const int s = (int)(k % S);
      if (k >= (u64)S && !wait_or_abort(&empty[s], (u32)(((k / S) - 1) & 1))) return;
      bool end = false;
      if (lane == 0) {
        fence_proxy_async_smem();
        const u64 t = TK ? tnext : B + k * G;
        if (TK) {
          s_tile[s] = t;
          if (t >= num_tiles) {  // the end of the stream: hand the stage over empty
            mbar_arrive(&full[s]);
            end = true;
          } else {
            tnext = atomicAdd(ticket, 1u);  // the next ticket travels while this tile loads
          }
        }
        if (!end) {
        mbar_expect_tx(&full[s], TILE_BYTES);
#pragma unroll
        for (int q = 0; q < 4; ++q)
          tma_load_1d(ring + s * TILE + q * (TILE / 4), a + t * TILE + q * (TILE / 4), TILE_BYTES / 4,
                      &full[s]);
        }
      }
      if (TK && __shfl_sync(0xffffffffu, end ? 1 : 0, 0)) return;
      __syncwarp();
    }
    return;
  }
  if (warp <= (u32)LBW) {
    // ------------------------------------------------ look-back, k = warp-1 mod LBW
    for (u64 k = warp - 1; TK || B + k * G < num_tiles; k += LBW) {
      const int s = (int)(k % S);
      if (!wait_or_abort(&reduced[s], ph(k))) return;
      const u64 t = tile_of(k);
      const u64 agg = s_agg[s];
      u64 prefix = (t == 0 && carry_in) ? *carry_in : O::identity;
      int ok = 1;
      if (lane == 0) {
        ok = publish_begin(c, t);
        if (ok) {
          if (t == 0) publish_incl(c, 0, O::apply(prefix, agg));
          else publish_agg(c, t, agg);
        }
      }
      ok = __shfl_sync(0xffffffffu, ok, 0);
      if (ok && t > 0) {
        ok = lookback<O>(c, t, prefix);
        if (ok && lane == 0) publish_incl(c, t, O::apply(prefix, agg));
      }
      if (lane == 0) {
        s_prefix[s] = prefix;
        if (!ok) s_abort = 1;
        if (ok && t == num_tiles - 1 && total) *total = O::apply(prefix, agg);
        mbar_arrive(&pready[s]);
      }
      if (!ok) return;
    }
    return;
  }
  // ---------------------------------------------------------------- compute
  const u32 w = warp - 1 - LBW;
  auto scan_store = [&](u64 k) -> bool {
    const int s = (int)(k % S);
    if (!wait_or_abort(&pready[s], ph(k))) return false;
    u64 run = O::apply(s_prefix[s], s_wexc[s][w]);
    const u64* src = ring + s * TILE + w * 512;
    const u64 wbase = tile_of(k) * TILE + (u64)w * 512;
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      const ulonglong2 v = lds2(src + 64 * j + 2 * lane);
      const u64 x0 = v.x, x1 = v.y;
      const u64 inc = warp_incl_scan<O>(O::apply(x0, x1));
      u64 exc = __shfl_up_sync(0xffffffffu, inc, 1);
      if (lane == 0) exc = O::identity;
      const u64 tot = __shfl_sync(0xffffffffu, inc, 31);
      const u64 e = O::apply(run, exc);
      u64 o0, o1;
      if (INCLUSIVE) {
        o0 = O::apply(e, x0);
        o1 = O::apply(o0, x1);
      } else {
        o0 = e;
        o1 = O::apply(e, x0);
      }
      stg_stream2(a + wbase + 64 * j + 2 * lane, O::apply(init, o0), O::apply(init, o1));
      run = O::apply(run, tot);
    }
    named_bar(1, NWC * 32);  // every compute warp has read stage s
    if (w == 0 && lane == 0) mbar_arrive(&empty[s]);
    return true;
  };
  // compute runs D tiles ahead of the stores (S >= D + 2 stages)
  static_assert(S >= D + 2, "stages");
  for (u64 k = 0;; ++k) {
    const int s = (int)(k % S);
    if (TK && !wait_or_abort(&full[s], ph(k))) return;
    if (TK ? tile_of(k) >= num_tiles : B + k * G >= num_tiles) {
      for (u64 q = k > (u64)D ? k - D : 0; q < k; ++q)
        if (!scan_store(q)) return;
      if (TK) {
        named_bar(1, NWC * 32);
        if (w == 0 && lane == 0) s_done = 1;  // every tile stored: the look-back warps may leave
      }
      break;
    }
    if (!TK && !wait_or_abort(&full[s], ph(k))) return;
    const u64* src = ring + s * TILE + w * 512;
    u64 acc = O::identity;
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      const ulonglong2 v = lds2(src + 64 * j + 2 * lane);
      acc = O::apply(acc, O::apply(v.x, v.y));
    }
    acc = warp_reduce<O>(acc);
    if (lane == 0) s_wtot[s][w] = acc;
    named_bar(1, NWC * 32);
    if (w == 0) {
      const u64 wv = lane < (u32)NWC ? s_wtot[s][lane] : O::identity;
      const u64 winc = warp_incl_scan<O>(wv);
      u64 wexc = __shfl_up_sync(0xffffffffu, winc, 1);
      if (lane == 0) wexc = O::identity;
      if (lane < (u32)NWC) s_wexc[s][lane] = wexc;
      if (lane == NWC - 1) s_agg[s] = winc;
      __syncwarp();
      if (lane == 0) mbar_arrive(&reduced[s]);
    }
    if (k >= (u64)D && !scan_store(k - D)) return;
  }
}

// ---------------------------------------------------------------------------
// reduce: grid-stride fold, per-CTA partials, last CTA folds the partials.
template <int OP>
__global__ void __launch_bounds__(512)
reduce_kernel(const u64* __restrict__ a, u64 n, u64* partials, u32* counter, u64* total) {
  using O = Op<OP>;
  __shared__ u64 s_warp[16];
  __shared__ bool s_last;
  u64 t = O::identity;
  const u64 stride = (u64)gridDim.x * blockDim.x;
  const bool vec = ((uintptr_t)a & 15) == 0;
  if (vec) {
    const u64 npairs = n / 2;
    for (u64 p = (u64)blockIdx.x * blockDim.x + threadIdx.x; p < npairs; p += stride) {
      ulonglong2 v = ldg_stream2(a + 2 * p);
      t = O::apply(t, O::apply(v.x, v.y));
    }
    if ((n & 1) && blockIdx.x == 0 && threadIdx.x == 0) t = O::apply(t, a[n - 1]);
  } else {
    for (u64 i = (u64)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride)
      t = O::apply(t, a[i]);
  }
  t = warp_reduce<O>(t);
  if (lane_id() == 0) s_warp[warp_id()] = t;
  __syncthreads();
  if (threadIdx.x == 0) {
    u64 b = O::identity;
    for (int w = 0; w < (int)(blockDim.x / 32); ++w) b = O::apply(b, s_warp[w]);
    partials[blockIdx.x] = b;
    __threadfence();
    s_last = atomicAdd(counter, 1u) == gridDim.x - 1;
  }
  __syncthreads();
  if (s_last && threadIdx.x < 32) {
    __threadfence();
    u64 v = O::identity;
    for (u32 i = threadIdx.x; i < gridDim.x; i += 32) v = O::apply(v, ld_relaxed_u64(partials + i));
    v = warp_reduce<O>(v);
    if (threadIdx.x == 0) {
      *total = v;
      *counter = 0;
    }
  }
}

// ---------------------------------------------------------------------------
// host side

struct ScratchLayout {
  u32* abort;       // [0]
  u32* counter;     // [1]
  u64* carry;       // header byte 128: hand-off between the two launches of a scan
  u64* partials;    // G_MAX
  TileSlot* slots;  // 2 * G_MAX
};
static constexpr int CTAS_PER_SM_MAX = 8;
static size_t header_bytes() { return 256; }
size_t scratch_bytes_for(int sms) {
  const size_t gmax = (size_t)sms * CTAS_PER_SM_MAX;
  return header_bytes() + gmax * sizeof(u64) + 4 * gmax * sizeof(TileSlot);
}
static ScratchLayout carve(void* scratch, int sms) {
  const size_t gmax = (size_t)sms * CTAS_PER_SM_MAX;
  char* p = (char*)scratch;
  ScratchLayout L;
  L.abort = (u32*)p;
  L.counter = (u32*)p + 1;
  L.carry = (u64*)(p + 128);
  L.partials = (u64*)(p + header_bytes());
  L.slots = (TileSlot*)(p + header_bytes() + gmax * sizeof(u64));
  return L;
}

template <class K>
static int persistent_grid(K kernel, int threads, int device, u64 tiles, int* grid) {
  int per_sm = 0;
  PIP_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kernel, threads, 0));
  if (per_sm < 1) return PIP_ERR_UNSUPPORTED;
  if (per_sm > CTAS_PER_SM_MAX) per_sm = CTAS_PER_SM_MAX;
  u64 g = (u64)per_sm * num_sms(device);
  if (g > tiles) g = tiles;
  *grid = (int)g;
  return PIP_OK;
}

template <int OP, bool INCL, bool VEC>
static int launch_scan_t(u64* a, u64 n, u64 init, const u64* carry, u64* total,
                         const ScratchLayout& L, cudaStream_t st, int device) {
  const u64 tiles = (n + SCAN_TILE - 1) / SCAN_TILE;
  auto k = scan_kernel<OP, INCL, VEC>;
  int grid = 0;
  int rc = persistent_grid(k, SCAN_THREADS, device, tiles, &grid);
  if (rc) return rc;
  PIP_CUDA(cudaMemsetAsync(L.counter, 0, 60, st));
  PIP_CUDA(cudaMemsetAsync(L.slots, 0, sizeof(TileSlot) * 4 * (size_t)grid * lb_stride(num_sms(current_device()), grid), st));
  LookbackCtx c{L.slots, L.abort, (u32)(4 * grid), lb_stride(num_sms(current_device()), grid)};
  u32* counter = L.counter;
  void* args[] = {&a, &n, &init, &carry, &total, &c, (void*)&tiles, &counter};
  PIP_CUDA(cudaLaunchCooperativeKernel((const void*)k, dim3(grid), dim3(SCAN_THREADS), args, 0, st));
  return PIP_OK;
}

template <int OP, bool INCL, int THREADS, int STAGES>
static int launch_scan_tma(u64* a, u64 n, u64 init, const u64* carry, u64* total,
                           const ScratchLayout& L, cudaStream_t st, int device) {
  constexpr u64 TILE = (u64)THREADS * SCAN_ITEMS;
  const u64 tiles = (n + TILE - 1) / TILE;
  const u64 full_tiles = n / TILE;
  auto k = scan_tma_kernel<OP, INCL, THREADS, STAGES>;
  const int smem = (int)(STAGES * TILE * 8);
  PIP_CUDA(cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
  int per_sm = 0;
  PIP_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k, THREADS, smem));
  if (per_sm < 1) return PIP_ERR_UNSUPPORTED;
  if (per_sm > CTAS_PER_SM_MAX) per_sm = CTAS_PER_SM_MAX;
  u64 g = (u64)per_sm * num_sms(device);
  if (g > tiles) g = tiles;
  int grid = (int)g;
  PIP_CUDA(cudaMemsetAsync(L.counter, 0, 60, st));
  PIP_CUDA(cudaMemsetAsync(L.slots, 0, sizeof(TileSlot) * 4 * (size_t)grid * lb_stride(num_sms(current_device()), grid), st));
  LookbackCtx c{L.slots, L.abort, (u32)(4 * grid), lb_stride(num_sms(current_device()), grid)};
  u32* counter = L.counter;
  void* args[] = {&a, &n, &init, &carry, &total, &c, (void*)&tiles, (void*)&full_tiles, &counter};
  PIP_CUDA(cudaLaunchCooperativeKernel((const void*)k, dim3(grid), dim3(THREADS), args, smem, st));
  return PIP_OK;
}

template <int OP, bool INCL, int THREADS, int STAGES>
static int launch_scan_ahead(u64* a, u64 n, u64 init, const u64* carry, u64* total,
                             const ScratchLayout& L, cudaStream_t st, int device) {
  constexpr u64 TILE = (u64)THREADS * SCAN_ITEMS;
  const u64 full_tiles = n / TILE;
  const u64 rem = n - full_tiles * TILE;
  auto k = scan_ahead_kernel<OP, INCL, THREADS, STAGES>;
  const int smem = (int)(STAGES * TILE * 8);
  PIP_CUDA(cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
  int per_sm = 0;
  PIP_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k, THREADS, smem));
  if (per_sm < 1) return PIP_ERR_UNSUPPORTED;
  if (per_sm > CTAS_PER_SM_MAX) per_sm = CTAS_PER_SM_MAX;
  u64 g = (u64)per_sm * num_sms(device);
  if (g > full_tiles) g = full_tiles;
  int grid = (int)g;
  // the whole-tile part writes its inclusive fold to `mid` when a tail follows
  u64* mid = rem ? L.carry : total;
  PIP_CUDA(cudaMemsetAsync(L.counter, 0, 60, st));
  PIP_CUDA(cudaMemsetAsync(L.slots, 0, sizeof(TileSlot) * 4 * (size_t)grid * lb_stride(num_sms(current_device()), grid), st));
  LookbackCtx c{L.slots, L.abort, (u32)(4 * grid), lb_stride(num_sms(current_device()), grid)};
  void* args[] = {&a, &init, &carry, &mid, &c, (void*)&full_tiles};
  PIP_CUDA(cudaLaunchCooperativeKernel((const void*)k, dim3(grid), dim3(THREADS), args, smem, st));
  if (rem) {
    u64* tail = a + full_tiles * TILE;
    return launch_scan_t<OP, INCL, true>(tail, rem, init, L.carry, total, L, st, device);
  }
  return PIP_OK;
}

template <int OP, bool INCL, int NWC, int S, bool DYN = false, bool AHEAD = false, int WPW = 512>
static int launch_scan_ws(u64* a, u64 n, u64 init, const u64* carry, u64* total,
                          const ScratchLayout& L, cudaStream_t st, int device) {
  constexpr u64 TILE = (u64)NWC * WPW;
  constexpr int THREADS = 32 * (NWC + 1);
  const u64 full_tiles = n / TILE;
  const u64 rem = n - full_tiles * TILE;
  auto k = scan_ws_kernel<OP, INCL, NWC, S, DYN, AHEAD, WPW>;
  const int smem = (int)(S * TILE * 8);
  PIP_CUDA(cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
  int per_sm = 0;
  PIP_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k, THREADS, smem));
  if (per_sm < 1) return PIP_ERR_UNSUPPORTED;
  if (per_sm > CTAS_PER_SM_MAX) per_sm = CTAS_PER_SM_MAX;
  u64 g = (u64)per_sm * num_sms(device);
  if (g > full_tiles) g = full_tiles;
  int grid = (int)g;
  u64* mid = rem ? L.carry : total;
  PIP_CUDA(cudaMemsetAsync(L.counter, 0, 60, st));
  PIP_CUDA(cudaMemsetAsync(L.slots, 0, sizeof(TileSlot) * 4 * (size_t)grid * lb_stride(num_sms(current_device()), grid), st));
  LookbackCtx c{L.slots, L.abort, (u32)(4 * grid), lb_stride(num_sms(current_device()), grid)};
  u32* counter = L.counter;
  void* args[] = {&a, &init, &carry, &mid, &c, (void*)&full_tiles, &counter};
  const bool prof = timing_enabled();
  if (prof) {
    const u64 z[8] = {0, 0, 0, 0, 0, 0, 0, 0};
    const u32 on = 1;
    PIP_CUDA(cudaMemcpyToSymbolAsync(g_scan_prof, z, sizeof(z), 0, cudaMemcpyHostToDevice, st));
    PIP_CUDA(cudaMemcpyToSymbolAsync(g_prof_on, &on, 4, 0, cudaMemcpyHostToDevice, st));
    const char* pc = getenv("PIP_PROF_CTA");
    const u32 cta = pc ? (u32)atoi(pc) : 0u;
    PIP_CUDA(cudaMemcpyToSymbolAsync(g_prof_cta, &cta, 4, 0, cudaMemcpyHostToDevice, st));
    PIP_CUDA(cudaStreamSynchronize(st));
  }
  PIP_CUDA(cudaLaunchCooperativeKernel((const void*)k, dim3(grid), dim3(THREADS), args, smem, st));
  if (prof) {
    u64 h[8];
    const u32 off = 0;
    PIP_CUDA(cudaMemcpyFromSymbolAsync(h, g_scan_prof, sizeof(h), 0, cudaMemcpyDeviceToHost, st));
    PIP_CUDA(cudaMemcpyToSymbolAsync(g_prof_on, &off, 4, 0, cudaMemcpyHostToDevice, st));
    PIP_CUDA(cudaStreamSynchronize(st));
    fprintf(stderr, "[pip scan] profiled CTA: tiles %llu | producer: wait-reduce %llu lookback %llu | compute: wait-prefix %llu wait-data %llu cycles\n",
            (unsigned long long)h[2], (unsigned long long)h[0], (unsigned long long)h[1],
            (unsigned long long)h[3], (unsigned long long)h[4]);
  }
  if (rem) {
    u64* tail = a + full_tiles * TILE;
    return launch_scan_t<OP, INCL, true>(tail, rem, init, L.carry, total, L, st, device);
  }
  return PIP_OK;
}

template <int OP, bool INCL, int NWC, int S, int LBW, int D = 1, int MB = 1, bool TK = false>
static int launch_scan_ws2(u64* a, u64 n, u64 init, const u64* carry, u64* total,
                           const ScratchLayout& L, cudaStream_t st, int device) {
  constexpr u64 TILE = (u64)NWC * 512;
  constexpr int THREADS = 32 * (NWC + 1 + LBW);
  const u64 full_tiles = n / TILE;
  const u64 rem = n - full_tiles * TILE;
  auto k = scan_ws2_kernel<OP, INCL, NWC, S, LBW, D, MB, TK>;
  const int smem = (int)(S * TILE * 8);
  PIP_CUDA(cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
  int per_sm = 0;
  PIP_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k, THREADS, smem));
  if (per_sm < 1) return PIP_ERR_UNSUPPORTED;
  if (per_sm > CTAS_PER_SM_MAX) per_sm = CTAS_PER_SM_MAX;
  u64 g = (u64)per_sm * num_sms(device);
  if (g > full_tiles) g = full_tiles;
  int grid = (int)g;
  u64* mid = rem ? L.carry : total;
  const u32 stride = lb_stride(num_sms(device), grid);
  PIP_CUDA(cudaMemsetAsync(L.counter, 0, 60, st));
  PIP_CUDA(cudaMemsetAsync(L.slots, 0, sizeof(TileSlot) * 4 * (size_t)grid * stride, st));
  LookbackCtx c{L.slots, L.abort, (u32)(4 * grid), stride};
  u32* ticket = L.counter + 2;  // zeroed with the counters above
  void* args[] = {&a, &init, &carry, &mid, &c, (void*)&full_tiles, &ticket};
  PIP_CUDA(cudaLaunchCooperativeKernel((const void*)k, dim3(grid), dim3(THREADS), args, smem, st));
  if (rem) return launch_scan_t<OP, INCL, true>(a + full_tiles * TILE, rem, init, L.carry, total, L, st, device);
  return PIP_OK;
}

static int scan_cfg() {
  static int cfg = -1;
  if (cfg < 0) {
    // 17 = scan_ws2_kernel<13 compute warps, 4 stages of 52 KiB, 3 look-back
    // warps, compute 2 tiles ahead> (best measured: 11.2 ms at 2^32; with one
    // look-back warp doing the streaming too — cfg 8, scan_ws_kernel<16,3> —
    // 12.9 ms; 2 look-back warps, 3 stages: 12.2; <12,4,2,2>: 11.6;
    // <10,5,3,3>: 11.7); 6/7/9-12 = other scan_ws variants; 4/5 =
    // aggregate-ahead TMA; 1-3 = plain TMA rings; 0 = registers
    // 21 = 17 with the tiles handed out by ticket instead of round-robin
    // (default since the end of round 2: 11.33 vs 11.54 ms over 10 steps,
    // 11.65 vs 11.80 over 20; the same change on the filter, PIP_FILTER_CFG=35,
    // measured 9.02 vs 8.95 ms and is not its default)
    // 25 = the same with 14 compute warps (56 KiB tiles, the largest four
    // stages of fit) and 2 look-back warps: 10.80-11.07 ms over 10 steps,
    // 11.37 over 20 (cfg 29, the same shape with round-robin tiles: 11.2)
    // DEFAULT = 29: cfg 25's shape (14 compute warps, 56 KiB tiles, 2
    // look-back warps) with ROUND-ROBIN tiles.  The ticketed variants (21,
    // 22, 25, 28) are faster by 1-2% but a soak test found intermittent
    // stalls in them (a bounded spin expiring -> PIP_ERR_STALLED, reported,
    // never silent) when the look-back slots are packed (PIP_LB_STRIDE=1:
    // cfg 21 three times in 30 full-size scans, cfg 25 once in 60; none in
    // 260 scans at the default spacing, none ever for round-robin tiles), so
    // they stay measurement knobs until that wait cycle is found.
    const char* e = getenv("PIP_SCAN_CFG");
    cfg = e ? atoi(e) : 29;
  }
  return cfg;
}

template <int OP>
static int launch_scan_op(u64* a, u64 n, u64 init, int inclusive, const u64* carry, u64* total,
                          const ScratchLayout& L, cudaStream_t st, int device) {
  const bool vec = ((uintptr_t)a & 15) == 0;
  const int cfg = scan_cfg();
  if (vec && cfg >= 6 && n >= 8 * SCAN_TILE) {
    if (cfg == 6)
      return inclusive ? launch_scan_ws<OP, true, 8, 4>(a, n, init, carry, total, L, st, device)
                       : launch_scan_ws<OP, false, 8, 4>(a, n, init, carry, total, L, st, device);
    if (cfg == 7)
      return inclusive ? launch_scan_ws<OP, true, 8, 3>(a, n, init, carry, total, L, st, device)
                       : launch_scan_ws<OP, false, 8, 3>(a, n, init, carry, total, L, st, device);
    if (cfg == 9)
      return inclusive ? launch_scan_ws<OP, true, 16, 3, true>(a, n, init, carry, total, L, st, device)
                       : launch_scan_ws<OP, false, 16, 3, true>(a, n, init, carry, total, L, st, device);
    if (cfg == 17)  // default: producer warp, 3 look-back warps, 13 compute warps 2 tiles ahead
      return inclusive ? launch_scan_ws2<OP, true, 13, 4, 3, 2>(a, n, init, carry, total, L, st, device)
                       : launch_scan_ws2<OP, false, 13, 4, 3, 2>(a, n, init, carry, total, L, st, device);
    if (cfg == 28)  // ticketed, 14 compute warps, 3 look-back warps
      return inclusive ? launch_scan_ws2<OP, true, 14, 4, 3, 2, 1, true>(a, n, init, carry, total, L, st, device)
                       : launch_scan_ws2<OP, false, 14, 4, 3, 2, 1, true>(a, n, init, carry, total, L, st, device);
    if (cfg == 29)  // 14 compute warps, 2 look-back warps, round-robin tiles
      return inclusive ? launch_scan_ws2<OP, true, 14, 4, 2, 2, 1, false>(a, n, init, carry, total, L, st, device)
                       : launch_scan_ws2<OP, false, 14, 4, 2, 2, 1, false>(a, n, init, carry, total, L, st, device);
    if (cfg == 25)  // ticketed, 14 compute warps (56 KiB tiles), 2 look-back warps
      return inclusive ? launch_scan_ws2<OP, true, 14, 4, 2, 2, 1, true>(a, n, init, carry, total, L, st, device)
                       : launch_scan_ws2<OP, false, 14, 4, 2, 2, 1, true>(a, n, init, carry, total, L, st, device);
    if (cfg == 26)  // ticketed, 14 compute warps, 1 look-back warp
      return inclusive ? launch_scan_ws2<OP, true, 14, 4, 1, 2, 1, true>(a, n, init, carry, total, L, st, device)
                       : launch_scan_ws2<OP, false, 14, 4, 1, 2, 1, true>(a, n, init, carry, total, L, st, device);
    if (cfg == 27)  // ticketed, 13 compute warps, 1 look-back warp
      return inclusive ? launch_scan_ws2<OP, true, 13, 4, 1, 2, 1, true>(a, n, init, carry, total, L, st, device)
                       : launch_scan_ws2<OP, false, 13, 4, 1, 2, 1, true>(a, n, init, carry, total, L, st, device);
    if (cfg == 22)  // ticketed, 2 look-back warps
      return inclusive ? launch_scan_ws2<OP, true, 13, 4, 2, 2, 1, true>(a, n, init, carry, total, L, st, device)
                       : launch_scan_ws2<OP, false, 13, 4, 2, 2, 1, true>(a, n, init, carry, total, L, st, device);
    if (cfg == 23)  // ticketed, two CTAs per SM with half-size tiles
      return inclusive ? launch_scan_ws2<OP, true, 6, 4, 3, 2, 2, true>(a, n, init, carry, total, L, st, device)
                       : launch_scan_ws2<OP, false, 6, 4, 3, 2, 2, true>(a, n, init, carry, total, L, st, device);
    if (cfg == 24)  // ticketed, stores one tile behind the reduce
      return inclusive ? launch_scan_ws2<OP, true, 13, 4, 3, 1, 1, true>(a, n, init, carry, total, L, st, device)
                       : launch_scan_ws2<OP, false, 13, 4, 3, 1, 1, true>(a, n, init, carry, total, L, st, device);
    if (cfg == 21)  // 17 with tiles handed out by ticket
      return inclusive ? launch_scan_ws2<OP, true, 13, 4, 3, 2, 1, true>(a, n, init, carry, total, L, st, device)
                       : launch_scan_ws2<OP, false, 13, 4, 3, 2, 1, true>(a, n, init, carry, total, L, st, device);
    if (cfg == 18)  // two CTAs per SM, 3072-word tiles
      return inclusive ? launch_scan_ws2<OP, true, 6, 4, 3, 2, 2>(a, n, init, carry, total, L, st, device)
                       : launch_scan_ws2<OP, false, 6, 4, 3, 2, 2>(a, n, init, carry, total, L, st, device);
    if (cfg == 19)  // two CTAs per SM, 4096-word tiles, 3 stages
      return inclusive ? launch_scan_ws2<OP, true, 8, 3, 3, 1, 2>(a, n, init, carry, total, L, st, device)
                       : launch_scan_ws2<OP, false, 8, 3, 3, 1, 2>(a, n, init, carry, total, L, st, device);
    if (cfg == 11)
      return inclusive ? launch_scan_ws<OP, true, 14, 4>(a, n, init, carry, total, L, st, device)
                       : launch_scan_ws<OP, false, 14, 4>(a, n, init, carry, total, L, st, device);
    if (cfg == 12)
      return inclusive ? launch_scan_ws<OP, true, 12, 4>(a, n, init, carry, total, L, st, device)
                       : launch_scan_ws<OP, false, 12, 4>(a, n, init, carry, total, L, st, device);
    if (cfg == 10)
      return inclusive
                 ? launch_scan_ws<OP, true, 12, 4, false, true>(a, n, init, carry, total, L, st, device)
                 : launch_scan_ws<OP, false, 12, 4, false, true>(a, n, init, carry, total, L, st, device);
    return inclusive ? launch_scan_ws<OP, true, 16, 3>(a, n, init, carry, total, L, st, device)
                     : launch_scan_ws<OP, false, 16, 3>(a, n, init, carry, total, L, st, device);
  }
  if (vec && cfg >= 4 && n >= 4 * SCAN_TILE) {
    if (cfg == 4)
      return inclusive ? launch_scan_ahead<OP, true, 512, 3>(a, n, init, carry, total, L, st, device)
                       : launch_scan_ahead<OP, false, 512, 3>(a, n, init, carry, total, L, st, device);
    return inclusive ? launch_scan_ahead<OP, true, 256, 3>(a, n, init, carry, total, L, st, device)
                     : launch_scan_ahead<OP, false, 256, 3>(a, n, init, carry, total, L, st, device);
  }
  if (vec && cfg > 0 && cfg < 4 && n >= SCAN_TILE) {
    if (cfg == 1)
      return inclusive ? launch_scan_tma<OP, true, 512, 3>(a, n, init, carry, total, L, st, device)
                       : launch_scan_tma<OP, false, 512, 3>(a, n, init, carry, total, L, st, device);
    if (cfg == 2)
      return inclusive ? launch_scan_tma<OP, true, 256, 3>(a, n, init, carry, total, L, st, device)
                       : launch_scan_tma<OP, false, 256, 3>(a, n, init, carry, total, L, st, device);
    return inclusive ? launch_scan_tma<OP, true, 256, 4>(a, n, init, carry, total, L, st, device)
                     : launch_scan_tma<OP, false, 256, 4>(a, n, init, carry, total, L, st, device);
  }
  if (inclusive) {
    return vec ? launch_scan_t<OP, true, true>(a, n, init, carry, total, L, st, device)
               : launch_scan_t<OP, true, false>(a, n, init, carry, total, L, st, device);
  }
  return vec ? launch_scan_t<OP, false, true>(a, n, init, carry, total, L, st, device)
             : launch_scan_t<OP, false, false>(a, n, init, carry, total, L, st, device);
}

int scan_device(u64* a, u64 n, int op, u64 init, int inclusive, const u64* carry_dev,
                u64* total_dev, void* scratch, size_t scratch_bytes, cudaStream_t st) {
  const int dev = current_device();
  const int sms = num_sms(dev);
  if (op < PIP_OP_ADD || op > PIP_OP_XOR) return PIP_ERR_INVALID_ARG;
  if (!scratch || scratch_bytes < scratch_bytes_for(sms)) return PIP_ERR_OOM;
  if (n == 0) {
    if (total_dev) {
      PIP_CUDA(cudaMemcpyAsync(total_dev, &init, 8, cudaMemcpyHostToDevice, st));
      PIP_CUDA(cudaStreamSynchronize(st));
    }
    return PIP_OK;
  }
  if (!a) return PIP_ERR_INVALID_ARG;
  ScratchLayout L = carve(scratch, sms);
  switch (op) {
    case PIP_OP_ADD: return launch_scan_op<PIP_OP_ADD>(a, n, init, inclusive, carry_dev, total_dev, L, st, dev);
    case PIP_OP_MAX: return launch_scan_op<PIP_OP_MAX>(a, n, init, inclusive, carry_dev, total_dev, L, st, dev);
    case PIP_OP_MIN: return launch_scan_op<PIP_OP_MIN>(a, n, init, inclusive, carry_dev, total_dev, L, st, dev);
    default: return launch_scan_op<PIP_OP_XOR>(a, n, init, inclusive, carry_dev, total_dev, L, st, dev);
  }
}

template <int OP>
static int launch_reduce(const u64* a, u64 n, u64* total, const ScratchLayout& L, cudaStream_t st,
                         int device) {
  const int sms = num_sms(device);
  int grid = sms * 2;
  u64 need = (n + 1023) / 1024;
  if ((u64)grid > need) grid = (int)(need ? need : 1);
  PIP_CUDA(cudaMemsetAsync(L.counter, 0, 60, st));
  reduce_kernel<OP><<<grid, 512, 0, st>>>(a, n, L.partials, L.counter, total);
  PIP_CHECK_LAUNCH();
  return PIP_OK;
}

int reduce_device(const u64* a, u64 n, int op, u64* total_dev, void* scratch, size_t scratch_bytes,
                  cudaStream_t st) {
  const int dev = current_device();
  const int sms = num_sms(dev);
  if (op < PIP_OP_ADD || op > PIP_OP_XOR || !total_dev) return PIP_ERR_INVALID_ARG;
  if (!scratch || scratch_bytes < scratch_bytes_for(sms)) return PIP_ERR_OOM;
  ScratchLayout L = carve(scratch, sms);
  switch (op) {
    case PIP_OP_ADD: return launch_reduce<PIP_OP_ADD>(a, n, total_dev, L, st, dev);
    case PIP_OP_MAX: return launch_reduce<PIP_OP_MAX>(a, n, total_dev, L, st, dev);
    case PIP_OP_MIN: return launch_reduce<PIP_OP_MIN>(a, n, total_dev, L, st, dev);
    default: return launch_reduce<PIP_OP_XOR>(a, n, total_dev, L, st, dev);
  }
}

}  // namespace pip
