// Stable in-place filter (strong.filter_kway, relaxed.filter_relaxed) and
// kept-count reduction.
//
// Reference: pkg/src/pipal/strong.py:283-349 — sqrt(n) chunks, a count
// pass, then batches of chunks whose destinations precede the batch's
// first source are compacted in parallel (:317-327); the predicate runs
// twice per element.  relaxed.py:284-309 retires one b(n)-prefix per round
// through a buffer.  Both leave a[0:m) = kept values in order, m returned,
// a[m:) unspecified.
//
// Here: ONE pass, predicate evaluated once.  Same persistent look-back
// skeleton as scan.cu with kept COUNTS as the scanned quantity.  In-place
// safety: a tile writes only to [prefix, prefix + kept) with prefix <= its
// own first index, i.e. into tiles that precede it; every such tile has
// published its aggregate — which it can only do after its loads returned —
// before this tile's look-back resolves.  So "destination precedes source"
// (the reference's batching rule, strong.py:317-327) holds at tile
// granularity without any batching.
#include <cstdlib>
#include "lookback.cuh"

namespace pip {

static constexpr int FILTER_THREADS = 512;
static constexpr u64 FILTER_TILE = (u64)FILTER_THREADS * 16;

int scan_grid_for(const void* kernel, int threads, int device, u64 tiles, int* grid);

// one tile with values + keep flags in registers: publish the kept count,
// look back for the output offset, scatter kept words (stable).  false => abort
template <int THREADS>
__device__ __forceinline__ bool filter_tile_body(const u64 (&x)[16], u32 keep, u64* __restrict__ a,
                                                 u64 tile, u64* m_out, const LookbackCtx& c,
                                                 u64 num_tiles, u64* s_warp, int* s_abort,
                                                 const u64* carry_in) {
  using O = Op<PIP_OP_ADD>;
  constexpr int NW = THREADS / 32;
  const u32 lane = lane_id(), warp = warp_id();
  const u32 lt = (1u << lane) - 1u;
  u64* s_ctl = s_warp + NW;     // [2]: agg, ok
  u64* s_lb = s_warp + NW + 2;  // block look-back scratch
  u64 cnt = warp_reduce<O>((u64)__popc(keep));
  if (lane == 0) s_warp[warp] = cnt;
  __syncthreads();
  if (warp == 0) {
    const u64 wv = lane < NW ? s_warp[lane] : 0;
    const u64 winc = warp_incl_scan<O>(wv);
    const u64 wexc = winc - wv;
    const u64 agg = __shfl_sync(0xffffffffu, winc, NW - 1);
    __syncwarp();
    if (lane < NW) s_warp[lane] = wexc;
    if (lane == 0) {
      const int ok = publish_begin(c, tile);
      if (ok) {
        // this tile's reads must be ordered before other tiles' writes into it
        __threadfence();
        if (tile == 0) publish_incl(c, tile, (carry_in ? *carry_in : 0) + agg);
        else publish_agg(c, tile, agg);
      }
      s_ctl[0] = agg;
      s_ctl[1] = ok;
    }
  }
  __syncthreads();
  const u64 agg = s_ctl[0];
  bool ok = s_ctl[1] != 0;
  u64 prefix = (tile == 0 && carry_in) ? *carry_in : 0;
  if (ok && tile > 0) {
    if (LB_BLOCK) {
      ok = block_lookback<O, THREADS>(c, tile, prefix, s_lb);
    } else {
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
    if (ok && threadIdx.x == 0) publish_incl(c, tile, prefix + agg);
  }
  if (!ok) {
    if (threadIdx.x == 0) atomicExch(c.abort, 1u);
    return false;
  }
  if (threadIdx.x == 0 && tile == num_tiles - 1 && m_out) *m_out = prefix + agg;
  (void)s_abort;
  u64 run = prefix + s_warp[warp];
#pragma unroll
  for (int j = 0; j < 8; ++j) {
    const bool f0 = (keep >> (2 * j)) & 1u, f1 = (keep >> (2 * j + 1)) & 1u;
    const u32 m0 = __ballot_sync(0xffffffffu, f0);
    const u32 m1 = __ballot_sync(0xffffffffu, f1);
    const u64 r0 = run + __popc(m0 & lt) + __popc(m1 & lt);
    if (f0) a[r0] = x[2 * j];
    if (f1) a[r0 + f0] = x[2 * j + 1];
    run += __popc(m0) + __popc(m1);
  }
  __syncthreads();
  return true;
}

template <bool VEC, int PC>
__global__ void __launch_bounds__(FILTER_THREADS, 2)
filter_kernel(u64* __restrict__ a, u64 n, DevPred p, u64* m_out, LookbackCtx c, u64 num_tiles,
              u32* counter, const u64* carry_in, u64* out) {
  __shared__ u64 s_warp[4 * (FILTER_THREADS / 32) + 4];
  __shared__ int s_abort;
  const u32 lane = lane_id(), warp = warp_id();
  (void)counter;
  for (u64 tile = blockIdx.x; tile < num_tiles; tile += gridDim.x) {
    const u64 wbase = tile * FILTER_TILE + (u64)warp * 512;
    const bool full = VEC && (tile * FILTER_TILE + FILTER_TILE <= n);
    u64 x[16];
    u32 keep = 0;
    if (full) {
#pragma unroll
      for (int j = 0; j < 8; ++j) {
        ulonglong2 v = ldg_stream2(a + wbase + 64 * j + 2 * lane);
        x[2 * j] = v.x;
        x[2 * j + 1] = v.y;
      }
#pragma unroll
      for (int k = 0; k < 16; ++k) keep |= (u32)pred_eval_t<PC>(p, x[k]) << k;
    } else {
#pragma unroll
      for (int j = 0; j < 8; ++j) {
        const u64 i0 = wbase + 64 * j + 2 * lane;
        x[2 * j] = i0 < n ? a[i0] : 0;
        x[2 * j + 1] = i0 + 1 < n ? a[i0 + 1] : 0;
        keep |= (u32)(i0 < n && pred_eval_t<PC>(p, x[2 * j])) << (2 * j);
        keep |= (u32)(i0 + 1 < n && pred_eval_t<PC>(p, x[2 * j + 1])) << (2 * j + 1);
      }
    }
    if (!filter_tile_body<FILTER_THREADS>(x, keep, out, tile, m_out, c, num_tiles, s_warp, &s_abort,
                                          carry_in))
      return;
  }
}

// runtime.compact_by_mask (runtime.py:335-355): the same look-back tile
// body with the keep flags read from a byte mask instead of a predicate
// (the reference's failure packing in detres.run_rounds, detres.py:303).
template <bool VEC>
__global__ void __launch_bounds__(FILTER_THREADS, 2)
compact_mask_kernel(u64* __restrict__ a, u64 n, const unsigned char* __restrict__ mask, u64* m_out,
                    LookbackCtx c, u64 num_tiles) {
  __shared__ u64 s_warp[4 * (FILTER_THREADS / 32) + 4];
  __shared__ int s_abort;
  const u32 lane = lane_id(), warp = warp_id();
  for (u64 tile = blockIdx.x; tile < num_tiles; tile += gridDim.x) {
    const u64 wbase = tile * FILTER_TILE + (u64)warp * 512;
    const bool full = VEC && (tile * FILTER_TILE + FILTER_TILE <= n);
    u64 x[16];
    u32 keep = 0;
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      const u64 i0 = wbase + 64 * j + 2 * lane;
      if (full) {
        const ulonglong2 v = ldg_stream2(a + wbase + 64 * j + 2 * lane);
        x[2 * j] = v.x;
        x[2 * j + 1] = v.y;
        const unsigned short mk = *(const unsigned short*)(mask + i0);
        keep |= (u32)((mk & 0xff) != 0) << (2 * j);
        keep |= (u32)((mk >> 8) != 0) << (2 * j + 1);
      } else {
        x[2 * j] = i0 < n ? a[i0] : 0;
        x[2 * j + 1] = i0 + 1 < n ? a[i0 + 1] : 0;
        keep |= (u32)(i0 < n && mask[i0] != 0) << (2 * j);
        keep |= (u32)(i0 + 1 < n && mask[i0 + 1] != 0) << (2 * j + 1);
      }
    }
    if (!filter_tile_body<FILTER_THREADS>(x, keep, a, tile, m_out, c, num_tiles, s_warp, &s_abort,
                                          nullptr))
      return;
  }
}

// TMA ring variant (16-byte aligned base), as scan_tma_kernel
template <int THREADS, int STAGES>
__global__ void __launch_bounds__(THREADS, 1)
filter_tma_kernel(u64* __restrict__ a, u64 n, DevPred p, u64* m_out, LookbackCtx c, u64 num_tiles,
                  u64 full_tiles, u32* counter) {
  constexpr u64 TILE = (u64)THREADS * 16;
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
  auto issue = [&](u64 k) {
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
    u64 x[16];
    u32 keep = 0;
    if (tile < full_tiles) {
      const u64* src = ring + s * TILE + warp * 512;
#pragma unroll
      for (int j = 0; j < 8; ++j) {
        const ulonglong2 v = lds2(src + 64 * j + 2 * lane);
        x[2 * j] = v.x;
        x[2 * j + 1] = v.y;
      }
#pragma unroll
      for (int q = 0; q < 16; ++q) keep |= (u32)pred_eval(p, x[q]) << q;
    } else {
      const u64 wbase = tile * TILE + (u64)warp * 512;
#pragma unroll
      for (int j = 0; j < 8; ++j) {
        const u64 i0 = wbase + 64 * j + 2 * lane;
        x[2 * j] = i0 < n ? a[i0] : 0;
        x[2 * j + 1] = i0 + 1 < n ? a[i0 + 1] : 0;
        keep |= (u32)(i0 < n && pred_eval(p, x[2 * j])) << (2 * j);
        keep |= (u32)(i0 + 1 < n && pred_eval(p, x[2 * j + 1])) << (2 * j + 1);
      }
    }
    __syncthreads();
    if (tid == 0) {
      fence_proxy_async_smem();
      issue(k + STAGES);
    }
    if (!filter_tile_body<THREADS>(x, keep, a, tile, m_out, c, num_tiles, s_warp, &s_abort, nullptr))
      return;
  }
}

// Aggregate-ahead pipeline (see scan_ahead_kernel in scan.cu): the next
// tile's kept count is published before this tile looks back, so the
// look-back never waits on a predecessor's HBM load.  In-place safety is
// unchanged: a tile publishes its count only after its data sits in shared
// memory, and writes only below its own end.
template <int THREADS, int STAGES>
__global__ void __launch_bounds__(THREADS, 1)
filter_ahead_kernel(u64* __restrict__ a, DevPred p, u64* m_out, LookbackCtx c, u64 num_tiles) {
  using O = Op<PIP_OP_ADD>;
  constexpr int NW = THREADS / 32;
  constexpr u64 TILE = (u64)THREADS * 16;
  constexpr u32 TILE_BYTES = (u32)(TILE * 8);
  extern __shared__ __align__(128) u64 ring[];
  __shared__ __align__(8) u64 bars[STAGES];
  __shared__ u64 s_wexc[STAGES][NW];
  __shared__ u64 s_agg[STAGES];
  __shared__ u64 s_tmp[NW + 4];
  const u32 tid = threadIdx.x, lane = lane_id(), warp = warp_id();
  const u32 lt = (1u << lane) - 1u;
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
  auto reduce_stage = [&](u64 k) {
    const int s = (int)(k % STAGES);
    mbar_wait(&bars[s], (u32)((k / STAGES) & 1));
    const u64* src = ring + s * TILE + warp * 512;
    u32 cnt = 0;
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      const ulonglong2 v = lds2(src + 64 * j + 2 * lane);
      cnt += (u32)pred_eval(p, v.x) + (u32)pred_eval(p, v.y);
    }
    const u64 t = warp_reduce<O>((u64)cnt);
    if (lane == 0) s_tmp[warp] = t;
    __syncthreads();
    if (warp == 0) {
      const u64 wv = lane < NW ? s_tmp[lane] : 0;
      const u64 winc = warp_incl_scan<O>(wv);
      if (lane < NW) s_wexc[s][lane] = winc - wv;
      if (lane == NW - 1) s_agg[s] = winc;
    }
    __syncthreads();
  };
  if (tid == 0)
    for (int k = 0; k < STAGES; ++k) issue(k);
  if ((u64)blockIdx.x >= num_tiles) return;
  reduce_stage(0);
  if (tid == 0) {
    const u64 t0 = blockIdx.x;
    const int ok = publish_begin(c, t0);
    if (ok) {
      if (t0 == 0) publish_incl(c, 0, s_agg[0]);
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
    if (tn < num_tiles) {
      reduce_stage(k + 1);
      if (tid == 0) {
        const int ok = publish_begin(c, tn);
        if (ok) publish_agg(c, tn, s_agg[(k + 1) % STAGES]);
        s_tmp[NW] = ok;
      }
    }
    if (warp == 0) {
      u64 prefix = 0;
      bool ok = true;
      if (tile > 0) {
        ok = lookback<O>(c, tile, prefix);
        if (ok && lane == 0) publish_incl(c, tile, prefix + s_agg[s]);
      }
      if (lane == 0) {
        s_tmp[NW + 1] = prefix;
        s_tmp[NW + 2] = ok;
        if (ok && tile == num_tiles - 1 && m_out) *m_out = prefix + s_agg[s];
      }
    }
    __syncthreads();
    if (!s_tmp[NW + 2] || (tn < num_tiles && !s_tmp[NW])) {
      if (tid == 0) atomicExch(c.abort, 1u);
      return;
    }
    u64 run = s_tmp[NW + 1] + s_wexc[s][warp];
    const u64* src = ring + s * TILE + warp * 512;
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      const ulonglong2 v = lds2(src + 64 * j + 2 * lane);
      const bool f0 = pred_eval(p, v.x), f1 = pred_eval(p, v.y);
      const u32 m0 = __ballot_sync(0xffffffffu, f0);
      const u32 m1 = __ballot_sync(0xffffffffu, f1);
      const u64 r0 = run + __popc(m0 & lt) + __popc(m1 & lt);
      if (f0) a[r0] = v.x;
      if (f1) a[r0 + f0] = v.y;
      run += __popc(m0) + __popc(m1);
    }
    __syncthreads();
    if (tid == 0) {
      fence_proxy_async_smem();
      issue(k + STAGES);
    }
  }
}

// Warp-specialized pipeline (see scan_ws_kernel in scan.cu): warp 0 streams
// tiles in with cp.async.bulk and runs publish / look-back for tile k while
// the compute warps count tile k (keeping each lane's keep bits) and scatter
// tile k-1.  The predicate runs once per word.  In-place safety is the same
// argument as above: a tile's count is published only after its words sit
// in shared memory, and a tile writes only below its own end.
template <int NWC, int S, int PC, bool DYN, bool AHEAD = false>
__global__ void __launch_bounds__(32 * (NWC + 1), 1)
filter_ws_kernel(u64* __restrict__ a, DevPred p, u64* m_out, LookbackCtx c, u64 num_tiles,
                 u32* counter) {
  using O = Op<PIP_OP_ADD>;
  constexpr u64 TILE = (u64)NWC * 512;
  constexpr u32 TILE_BYTES = (u32)(TILE * 8);
  constexpr u64 STRIDE = TILE + 2;  // + 2 words: the compacted output may start one word in
  extern __shared__ __align__(128) u64 ring[];
  __shared__ __align__(8) u64 full[S], reduced[S], pready[S], empty[S];
  __shared__ u64 s_wtot[S][NWC];
  __shared__ u64 s_wexc[S][NWC];
  __shared__ u64 s_agg[S];
  __shared__ u64 s_prefix[S];
  __shared__ u32 s_keep[S][NWC * 32];
  __shared__ int s_abort;
  __shared__ u64 s_tile[S];  // DYN: tile id of each stage (claimed at issue)
  const u32 tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const u32 lt = (1u << lane) - 1u;
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
  auto issue = [&](u64 k) {
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
      tma_load_1d(ring + s * STRIDE + q * (TILE / 4), a + t * TILE + q * (TILE / 4), TILE_BYTES / 4,
                  &full[s]);
  };
  if (warp == 0) {
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
            if (okn) { __threadfence(); publish_agg(c, tn, s_agg[sn]); };
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
      mbar_wait(&reduced[s], (u32)((k / S) & 1));
      const u64 agg = s_agg[s];
      u64 prefix = 0;
      int ok = 1;
      if (lane == 0 && (!AHEAD || k == 0)) {
        ok = publish_begin(c, t);
        if (ok) {
          __threadfence();
          if (t == 0) publish_incl(c, 0, agg);
          else publish_agg(c, t, agg);
        }
      }
      ok = __shfl_sync(0xffffffffu, ok, 0);
      if (ok && t > 0) {
        ok = lookback<O>(c, t, prefix);
        if (ok && lane == 0) publish_incl(c, t, prefix + agg);
      }
      if (lane == 0) {
        s_prefix[s] = prefix;
        if (!ok) s_abort = 1;
        if (ok && t == num_tiles - 1 && m_out) *m_out = prefix + agg;
        mbar_arrive(&pready[s]);
      }
      if (!ok) return;
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
  const u32 w = warp - 1;
  // scatter: the kept words of the tile are compacted inside its own stage
  // buffer (every warp first pulls its 16 words per lane into registers) and
  // leave with one bulk store; only <= 2 ragged words go through the LSU
  auto scatter = [&](u64 k) -> bool {
    const int s = (int)(k % S);
    mbar_wait(&pready[s], (u32)((k / S) & 1));
    if (s_abort) return false;
    const u64 prefix = s_prefix[s];
    const u64 agg = s_agg[s];
    u64* stage = ring + s * STRIDE;
    // word parity of the destination: compacted word q sits at stage[par + q]
    // so that shared and global addresses agree modulo 16 bytes
    const u32 par = (u32)(((uintptr_t)(a + prefix) >> 3) & 1u);
    u32 run = (u32)s_wexc[s][w] + par;
    const u32 keep = s_keep[s][w * 32 + lane];
    const u64* src = stage + w * 512;
    u64 vx[8], vy[8];
    u32 pos[8];
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      const bool f0 = (keep >> (2 * j)) & 1u, f1 = (keep >> (2 * j + 1)) & 1u;
      const u32 m0 = __ballot_sync(0xffffffffu, f0);
      const u32 m1 = __ballot_sync(0xffffffffu, f1);
      pos[j] = run + __popc(m0 & lt) + __popc(m1 & lt);
      const ulonglong2 v = lds2(src + 64 * j + 2 * lane);
      vx[j] = v.x;
      vy[j] = v.y;
      run += __popc(m0) + __popc(m1);
    }
    named_bar(1, NWC * 32);  // the whole tile is in registers
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      const bool f0 = (keep >> (2 * j)) & 1u, f1 = (keep >> (2 * j + 1)) & 1u;
      if (f0) stage[pos[j]] = vx[j];
      if (f1) stage[pos[j] + (f0 ? 1u : 0u)] = vy[j];
    }
    fence_proxy_async_smem();
    named_bar(1, NWC * 32);
    if (w == 0 && lane == 0) {
      const u32 head = par && agg ? 1u : 0u;
      const u32 body = (u32)((agg - head) & ~1ull);
      if (head) a[prefix] = stage[1];
      if (head + body < agg) a[prefix + agg - 1] = stage[par + agg - 1];
      if (body) {
        tma_store_1d(a + prefix + head, stage + par + head, body * 8u);
        bulk_commit();
        bulk_wait_read_all();  // the stage may be refilled once the store has read it
      }
      mbar_arrive(&empty[s]);
    }
    return true;
  };
  auto reduce_tile = [&](u64 k) {
    const int s = (int)(k % S);
    mbar_wait(&full[s], (u32)((k / S) & 1));
    const u64* src = ring + s * STRIDE + w * 512;
    u32 keep = 0;
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      const ulonglong2 v = lds2(src + 64 * j + 2 * lane);
      keep |= ((u32)pred_eval_t<PC>(p, v.x) << (2 * j)) | ((u32)pred_eval_t<PC>(p, v.y) << (2 * j + 1));
    }
    s_keep[s][w * 32 + lane] = keep;
    const u64 cnt = warp_reduce<O>((u64)__popc(keep));
    if (lane == 0) s_wtot[s][w] = cnt;
    named_bar(1, NWC * 32);
    if (w == 0) {
      const u64 wv = lane < (u32)NWC ? s_wtot[s][lane] : 0;
      const u64 winc = warp_incl_scan<O>(wv);
      if (lane < (u32)NWC) s_wexc[s][lane] = winc - wv;
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
      if (!scatter(k)) return;
      if (B + (k + 2) * G < num_tiles) reduce_tile(k + 2);
    }
    if (w == 0 && lane == 0) bulk_wait_all();
    return;
  }
  for (u64 k = 0;; ++k) {
    const int s = (int)(k % S);
    if (DYN) mbar_wait(&full[s], (u32)((k / S) & 1));
    const u64 t = DYN ? s_tile[s] : B + k * G;
    if (t >= num_tiles) {
      if (k > 0) scatter(k - 1);
      if (w == 0 && lane == 0) bulk_wait_all();  // the bulk stores have landed
      break;
    }
    if (!DYN) mbar_wait(&full[s], (u32)((k / S) & 1));
    const u64* src = ring + s * STRIDE + w * 512;
    u32 keep = 0;
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      const ulonglong2 v = lds2(src + 64 * j + 2 * lane);
      keep |= ((u32)pred_eval_t<PC>(p, v.x) << (2 * j)) | ((u32)pred_eval_t<PC>(p, v.y) << (2 * j + 1));
    }
    s_keep[s][w * 32 + lane] = keep;
    const u64 cnt = warp_reduce<O>((u64)__popc(keep));
    if (lane == 0) s_wtot[s][w] = cnt;
    named_bar(1, NWC * 32);
    if (w == 0) {
      const u64 wv = lane < (u32)NWC ? s_wtot[s][lane] : 0;
      const u64 winc = warp_incl_scan<O>(wv);
      if (lane < (u32)NWC) s_wexc[s][lane] = winc - wv;
      if (lane == NWC - 1) s_agg[s] = winc;
      __syncwarp();
      if (lane == 0) mbar_arrive(&reduced[s]);
    }
    if (k > 0 && !scatter(k - 1)) return;
  }
}

// Split-role pipeline (see scan_ws2_kernel): warp 0 streams tiles in, LBW
// look-back warps take tiles round-robin so consecutive look-backs overlap,
// NWC compute warps count tile k and compact + store tile k - D.
// TK: tiles handed out by ticket instead of round-robin (see scan_ws2_kernel).
// BLK: each lane owns 16 CONSECUTIVE words of its warp's 1024 (read at a lane
// rotation, so the 16-byte shared-memory loads stay conflict-free): a kept
// word's place is the lane's base (one 5-step warp scan of the lane counts)
// plus the kept words below it in the lane's own mask -- no ballots.
template <int NWC, int S, int PC, int LBW, int D, int J, int MB = 1, bool TK = false, bool BLK = false>
__global__ void __launch_bounds__(32 * (NWC + 1 + LBW), MB)
filter_ws2_kernel(u64* __restrict__ a, DevPred p, u64* m_out, LookbackCtx c, u64 num_tiles,
                  u32* ticket) {
  using O = Op<PIP_OP_ADD>;
  constexpr u64 TILE = (u64)NWC * 64 * J;  // J word pairs per lane
  constexpr u32 TILE_BYTES = (u32)(TILE * 8);
  constexpr u64 STRIDE = TILE + 2;  // + 2 words: the compacted output may start one word in
  static_assert(S >= D + 2, "stages");
  static_assert(J >= 1 && J <= 8, "keep bits fit a u32");
  extern __shared__ __align__(128) u64 ring[];
  __shared__ __align__(8) u64 full[S], reduced[S], pready[S], empty[S];
  __shared__ u64 s_wtot[S][NWC];
  __shared__ u64 s_wexc[S][NWC];
  __shared__ u64 s_agg[S];
  __shared__ u64 s_prefix[S];
  // (each lane's keep bits of the tiles between count and compaction stay in
  // its registers: the same lane compacts the words it counted)
  __shared__ volatile int s_abort;
  __shared__ volatile u64 s_tile[S];  // TK: the tile in each stage (>= num_tiles: the stream's end)
  __shared__ volatile int s_done;     // TK: every tile of this CTA is stored; look-back warps leave
  const u32 tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const u32 lt = (1u << lane) - 1u;
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
          tma_load_1d(ring + s * STRIDE + q * (TILE / 4), a + t * TILE + q * (TILE / 4), TILE_BYTES / 4,
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
      u64 prefix = 0;
      int ok = 1;
      if (lane == 0) {
        ok = publish_begin(c, t);
        if (ok) {  // (the tile's bulk reads completed before it was reduced)
          if (t == 0) publish_incl(c, 0, agg);
          else publish_agg(c, t, agg);
        }
      }
      ok = __shfl_sync(0xffffffffu, ok, 0);
      if (ok && t > 0) {
        ok = lookback<O>(c, t, prefix);
        if (ok && lane == 0) publish_incl(c, t, prefix + agg);
      }
      if (lane == 0) {
        s_prefix[s] = prefix;
        if (!ok) s_abort = 1;
        if (ok && t == num_tiles - 1 && m_out) *m_out = prefix + agg;
        mbar_arrive(&pready[s]);
      }
      if (!ok) return;
    }
    return;
  }
  // ---------------------------------------------------------------- compute
  const u32 w = warp - 1 - LBW;
  // the kept words of a tile are compacted inside its own stage buffer (every
  // warp first pulls its 16 words per lane into registers) and leave with one
  // bulk store; only <= 2 ragged words go through the LSU
  auto scatter = [&](u64 k, const u32 keep) -> bool {
    const int s = (int)(k % S);
    if (!wait_or_abort(&pready[s], ph(k))) return false;
    const u64 prefix = s_prefix[s];
    const u64 agg = s_agg[s];
    u64* stage = ring + s * STRIDE;
    // word parity of the destination: compacted word q sits at stage[par + q]
    // so that shared and global addresses agree modulo 16 bytes
    const u32 par = (u32)(((uintptr_t)(a + prefix) >> 3) & 1u);
    u32 run = (u32)s_wexc[s][w] + par;
    const u64* src = stage + w * (64 * J);
    u64 vx[J], vy[J];
    u32 pos[J];
    if (BLK) {
      const u32 cl = __popc(keep);
      u32 inc = cl;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const u32 t = __shfl_up_sync(0xffffffffu, inc, o);
        if (lane >= (u32)o) inc += t;
      }
      run += inc - cl;  // the lane's first kept word
#pragma unroll
      for (int j = 0; j < J; ++j) {
        const u32 pj = ((u32)j + lane) & (J - 1);
        const ulonglong2 v = lds2(src + 2 * J * lane + 2 * pj);
        vx[j] = v.x;
        vy[j] = v.y;
      }
    } else {
#pragma unroll
    for (int j = 0; j < J; ++j) {
      const bool f0 = (keep >> (2 * j)) & 1u, f1 = (keep >> (2 * j + 1)) & 1u;
      const u32 m0 = __ballot_sync(0xffffffffu, f0);
      const u32 m1 = __ballot_sync(0xffffffffu, f1);
      pos[j] = run + __popc(m0 & lt) + __popc(m1 & lt);
      const ulonglong2 v = lds2(src + 64 * j + 2 * lane);
      vx[j] = v.x;
      vy[j] = v.y;
      run += __popc(m0) + __popc(m1);
    }
    }
    named_bar(1, NWC * 32);  // the whole tile is in registers
    if (BLK) {
#pragma unroll
      for (int j = 0; j < J; ++j) {
        const u32 b0 = 2 * (((u32)j + lane) & (J - 1));
        const bool f0 = (keep >> b0) & 1u, f1 = (keep >> (b0 + 1)) & 1u;
        const u32 at = run + __popc(keep & ((1u << b0) - 1u));
        if (f0) stage[at] = vx[j];
        if (f1) stage[at + (f0 ? 1u : 0u)] = vy[j];
      }
    } else {
#pragma unroll
    for (int j = 0; j < J; ++j) {
      const bool f0 = (keep >> (2 * j)) & 1u, f1 = (keep >> (2 * j + 1)) & 1u;
      if (f0) stage[pos[j]] = vx[j];
      if (f1) stage[pos[j] + (f0 ? 1u : 0u)] = vy[j];
    }
    }
    fence_proxy_async_smem();
    named_bar(1, NWC * 32);
    if (w == 0 && lane == 0) {
      const u32 head = par && agg ? 1u : 0u;
      const u32 body = (u32)((agg - head) & ~1ull);
      if (head) a[prefix] = stage[1];
      if (head + body < agg) a[prefix + agg - 1] = stage[par + agg - 1];
      if (body) {
        tma_store_1d(a + prefix + head, stage + par + head, body * 8u);
        bulk_commit();
        bulk_wait_read_all();  // the stage may be refilled once the store has read it
      }
      mbar_arrive(&empty[s]);
    }
    return true;
  };
  u32 kq[D + 1];  // kq[j]: keep bits of tile k - j
#pragma unroll
  for (int j = 0; j <= D; ++j) kq[j] = 0;
  for (u64 k = 0;; ++k) {
    const int s = (int)(k % S);
    if (TK && !wait_or_abort(&full[s], ph(k))) break;
    if (TK ? tile_of(k) >= num_tiles : B + k * G >= num_tiles) {
      // the last D tiles (fewer at the start): tile k - j counted j steps ago
#pragma unroll
      for (int j = D; j >= 1; --j)
        if (k >= (u64)j && !scatter(k - j, kq[j - 1])) break;
      if (TK) {
        named_bar(1, NWC * 32);
        if (w == 0 && lane == 0) s_done = 1;  // every tile stored: the look-back warps may leave
      }
      break;
    }
    if (!TK && !wait_or_abort(&full[s], ph(k))) break;
    const u64* src = ring + s * STRIDE + w * (64 * J);
    u32 keep = 0;
    if (BLK) {
      static_assert(!BLK || (J & (J - 1)) == 0, "lane rotation needs a power-of-two J");
#pragma unroll
      for (int j = 0; j < J; ++j) {
        const u32 pj = ((u32)j + lane) & (J - 1);
        const ulonglong2 v = lds2(src + 2 * J * lane + 2 * pj);
        keep |= ((u32)pred_raw_t<PC>(p, v.x) << (2 * pj)) | ((u32)pred_raw_t<PC>(p, v.y) << (2 * pj + 1));
      }
    } else {
#pragma unroll
    for (int j = 0; j < J; ++j) {
      const ulonglong2 v = lds2(src + 64 * j + 2 * lane);
      keep |= ((u32)pred_raw_t<PC>(p, v.x) << (2 * j)) | ((u32)pred_raw_t<PC>(p, v.y) << (2 * j + 1));
    }
    }
    if (PC != PC_GEN && p.negate) keep ^= (2 * J >= 32) ? 0xffffffffu : ((1u << (2 * J)) - 1u);
#pragma unroll
    for (int j = D; j >= 1; --j) kq[j] = kq[j - 1];
    kq[0] = keep;
    const u64 cnt = __reduce_add_sync(0xffffffffu, (u32)__popc(keep));  // one REDUX, not 10 shuffles
    if (lane == 0) s_wtot[s][w] = cnt;
    named_bar(1, NWC * 32);
    if (w == 0) {
      // tile counts fit 32 bits: a 32-bit shuffle scan (5 shuffles, not 10)
      const u32 wv = lane < (u32)NWC ? (u32)s_wtot[s][lane] : 0u;
      u32 winc = wv;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const u32 t = __shfl_up_sync(0xffffffffu, winc, o);
        if (lane >= (u32)o) winc += t;
      }
      if (lane < (u32)NWC) s_wexc[s][lane] = winc - wv;
      if (lane == NWC - 1) s_agg[s] = winc;
      __syncwarp();
      if (lane == 0) mbar_arrive(&reduced[s]);
    }
    if (k >= (u64)D && !scatter(k - D, kq[D])) break;
  }
  if (w == 0 && lane == 0) bulk_wait_all();  // the bulk stores have landed
}

template <int PC>
__global__ void __launch_bounds__(512)
count_kernel(const u64* __restrict__ a, u64 n, DevPred p, u64* partials, u32* counter, u64* total) {
  __shared__ u64 s_warp[16];
  __shared__ bool s_last;
  u64 t = 0;
  const u64 stride = (u64)gridDim.x * blockDim.x;
  const bool vec = ((uintptr_t)a & 15) == 0;
  if (vec) {
    const u64 npairs = n / 2;
#pragma unroll 4
    for (u64 q = (u64)blockIdx.x * blockDim.x + threadIdx.x; q < npairs; q += stride) {
      ulonglong2 v = ldg_stream2(a + 2 * q);
      t += (u64)pred_eval_t<PC>(p, v.x) + (u64)pred_eval_t<PC>(p, v.y);
    }
    if ((n & 1) && blockIdx.x == 0 && threadIdx.x == 0) t += pred_eval_t<PC>(p, a[n - 1]);
  } else {
    for (u64 i = (u64)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride)
      t += pred_eval_t<PC>(p, a[i]);
  }
  t = warp_reduce<Op<PIP_OP_ADD>>(t);
  if (lane_id() == 0) s_warp[warp_id()] = t;
  __syncthreads();
  if (threadIdx.x == 0) {
    u64 b = 0;
    for (int w = 0; w < (int)(blockDim.x / 32); ++w) b += s_warp[w];
    partials[blockIdx.x] = b;
    __threadfence();
    s_last = atomicAdd(counter, 1u) == gridDim.x - 1;
  }
  __syncthreads();
  if (s_last && threadIdx.x < 32) {
    __threadfence();
    u64 v = 0;
    for (u32 i = threadIdx.x; i < gridDim.x; i += 32) v += ld_relaxed_u64(partials + i);
    v = warp_reduce<Op<PIP_OP_ADD>>(v);
    if (threadIdx.x == 0) {
      *total = v;
      *counter = 0;
    }
  }
}

// ---------------------------------------------------------------------------
// host

struct ScratchLayoutF {
  u32* abort;
  u32* counter;
  u64* carry;
  u64* partials;
  TileSlot* slots;
};
size_t scratch_bytes_for(int sms);
static ScratchLayoutF carve_f(void* scratch, int sms) {
  const size_t gmax = (size_t)sms * 8;
  char* p = (char*)scratch;
  ScratchLayoutF L;
  L.abort = (u32*)p;
  L.counter = (u32*)p + 1;
  L.carry = (u64*)(p + 128);
  L.partials = (u64*)(p + 256);
  L.slots = (TileSlot*)(p + 256 + gmax * sizeof(u64));
  return L;
}

static int pred_class(const DevPred& p) {
  if (p.kind == PIP_PRED_MASK_EQ) return PC_MASK;
  if (p.kind == PIP_PRED_MOD_EQ) return p.tz == 0 ? (p.b == 0 ? PC_MODODD0 : PC_MODODD) : PC_MOD;
  return PC_GEN;
}

template <bool VEC, int PC>
static int launch_filter_pc(u64* a, u64 n, const DevPred& p, u64* m_dev, const ScratchLayoutF& L,
                            cudaStream_t st, int dev, const u64* carry_in, u64* out);

template <bool VEC>
static int launch_filter(u64* a, u64 n, const DevPred& p, u64* m_dev, const ScratchLayoutF& L,
                         cudaStream_t st, int dev, const u64* carry_in = nullptr,
                         u64* out = nullptr) {
  if (!out) out = a;
  switch (pred_class(p)) {
    case PC_MASK: return launch_filter_pc<VEC, PC_MASK>(a, n, p, m_dev, L, st, dev, carry_in, out);
    case PC_MOD: return launch_filter_pc<VEC, PC_MOD>(a, n, p, m_dev, L, st, dev, carry_in, out);
    case PC_MODODD: return launch_filter_pc<VEC, PC_MODODD>(a, n, p, m_dev, L, st, dev, carry_in, out);
    case PC_MODODD0: return launch_filter_pc<VEC, PC_MODODD0>(a, n, p, m_dev, L, st, dev, carry_in, out);
    default: return launch_filter_pc<VEC, PC_GEN>(a, n, p, m_dev, L, st, dev, carry_in, out);
  }
}

template <bool VEC, int PC>
static int launch_filter_pc(u64* a, u64 n, const DevPred& p, u64* m_dev, const ScratchLayoutF& L,
                            cudaStream_t st, int dev, const u64* carry_in, u64* out) {
  const u64 tiles = (n + FILTER_TILE - 1) / FILTER_TILE;
  auto k = filter_kernel<VEC, PC>;
  int per_sm = 0;
  PIP_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k, FILTER_THREADS, 0));
  if (per_sm < 1) return PIP_ERR_UNSUPPORTED;
  if (per_sm > 8) per_sm = 8;
  u64 g = (u64)per_sm * num_sms(dev);
  if (g > tiles) g = tiles;
  int grid = (int)g;
  PIP_CUDA(cudaMemsetAsync(L.counter, 0, 60, st));
  PIP_CUDA(cudaMemsetAsync(L.slots, 0, sizeof(TileSlot) * 4 * (size_t)grid * lb_stride(num_sms(current_device()), grid), st));
  LookbackCtx c{L.slots, L.abort, (u32)(4 * grid), lb_stride(num_sms(current_device()), grid)};
  DevPred pp = p;
  u32* counter = L.counter;
  void* args[] = {&a, &n, &pp, &m_dev, &c, (void*)&tiles, &counter, &carry_in, &out};
  PIP_CUDA(cudaLaunchCooperativeKernel((const void*)k, dim3(grid), dim3(FILTER_THREADS), args, 0, st));
  return PIP_OK;
}

template <int THREADS, int STAGES>
static int launch_filter_tma(u64* a, u64 n, const DevPred& p, u64* m_dev, const ScratchLayoutF& L,
                             cudaStream_t st, int dev) {
  constexpr u64 TILE = (u64)THREADS * 16;
  const u64 tiles = (n + TILE - 1) / TILE, full_tiles = n / TILE;
  auto k = filter_tma_kernel<THREADS, STAGES>;
  const int smem = (int)(STAGES * TILE * 8);
  PIP_CUDA(cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
  int per_sm = 0;
  PIP_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k, THREADS, smem));
  if (per_sm < 1) return PIP_ERR_UNSUPPORTED;
  if (per_sm > 8) per_sm = 8;
  u64 g = (u64)per_sm * num_sms(dev);
  if (g > tiles) g = tiles;
  int grid = (int)g;
  PIP_CUDA(cudaMemsetAsync(L.counter, 0, 60, st));
  PIP_CUDA(cudaMemsetAsync(L.slots, 0, sizeof(TileSlot) * 4 * (size_t)grid * lb_stride(num_sms(current_device()), grid), st));
  LookbackCtx c{L.slots, L.abort, (u32)(4 * grid), lb_stride(num_sms(current_device()), grid)};
  DevPred pp = p;
  u32* counter = L.counter;
  void* args[] = {&a, &n, &pp, &m_dev, &c, (void*)&tiles, (void*)&full_tiles, &counter};
  PIP_CUDA(cudaLaunchCooperativeKernel((const void*)k, dim3(grid), dim3(THREADS), args, smem, st));
  return PIP_OK;
}

template <int THREADS, int STAGES>
static int launch_filter_ahead(u64* a, u64 n, const DevPred& p, u64* m_dev,
                               const ScratchLayoutF& L, cudaStream_t st, int dev) {
  constexpr u64 TILE = (u64)THREADS * 16;
  const u64 full_tiles = n / TILE, rem = n - full_tiles * TILE;
  auto k = filter_ahead_kernel<THREADS, STAGES>;
  const int smem = (int)(STAGES * TILE * 8);
  PIP_CUDA(cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
  int per_sm = 0;
  PIP_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k, THREADS, smem));
  if (per_sm < 1) return PIP_ERR_UNSUPPORTED;
  if (per_sm > 8) per_sm = 8;
  u64 g = (u64)per_sm * num_sms(dev);
  if (g > full_tiles) g = full_tiles;
  int grid = (int)g;
  u64* mid = rem ? L.carry : m_dev;
  PIP_CUDA(cudaMemsetAsync(L.counter, 0, 60, st));
  PIP_CUDA(cudaMemsetAsync(L.slots, 0, sizeof(TileSlot) * 4 * (size_t)grid * lb_stride(num_sms(current_device()), grid), st));
  LookbackCtx c{L.slots, L.abort, (u32)(4 * grid), lb_stride(num_sms(current_device()), grid)};
  DevPred pp = p;
  void* args[] = {&a, &pp, &mid, &c, (void*)&full_tiles};
  PIP_CUDA(cudaLaunchCooperativeKernel((const void*)k, dim3(grid), dim3(THREADS), args, smem, st));
  if (rem) {
    // tail: kept words continue at a[m_full ...]; the tail sits 16-byte aligned
    return launch_filter<true>(a + full_tiles * TILE, rem, p, m_dev, L, st, dev, L.carry, a);
  }
  return PIP_OK;
}

template <int NWC, int S, int PC, bool DYN, bool AHEAD = false>
static int launch_filter_ws_pc(u64* a, u64 n, const DevPred& p, u64* m_dev,
                               const ScratchLayoutF& L, cudaStream_t st, int dev) {
  constexpr u64 TILE = (u64)NWC * 512;
  constexpr int THREADS = 32 * (NWC + 1);
  const u64 full_tiles = n / TILE, rem = n - full_tiles * TILE;
  auto k = filter_ws_kernel<NWC, S, PC, DYN, AHEAD>;
  const int smem = (int)(S * (TILE + 2) * 8);
  PIP_CUDA(cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
  int per_sm = 0;
  PIP_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k, THREADS, smem));
  if (per_sm < 1) return PIP_ERR_UNSUPPORTED;
  if (per_sm > 8) per_sm = 8;
  u64 g = (u64)per_sm * num_sms(dev);
  if (g > full_tiles) g = full_tiles;
  int grid = (int)g;
  u64* mid = rem ? L.carry : m_dev;
  PIP_CUDA(cudaMemsetAsync(L.counter, 0, 60, st));
  PIP_CUDA(cudaMemsetAsync(L.slots, 0, sizeof(TileSlot) * 4 * (size_t)grid * lb_stride(num_sms(current_device()), grid), st));
  LookbackCtx c{L.slots, L.abort, (u32)(4 * grid), lb_stride(num_sms(current_device()), grid)};
  DevPred pp = p;
  u32* counter = L.counter;
  void* args[] = {&a, &pp, &mid, &c, (void*)&full_tiles, &counter};
  PIP_CUDA(cudaLaunchCooperativeKernel((const void*)k, dim3(grid), dim3(THREADS), args, smem, st));
  if (rem) return launch_filter<true>(a + full_tiles * TILE, rem, p, m_dev, L, st, dev, L.carry, a);
  return PIP_OK;
}

template <int NWC, int S, int PC, int LBW, int D, int J, int MB = 1, bool TK = false, bool BLK = false>
static int launch_filter_ws2_pc(u64* a, u64 n, const DevPred& p, u64* m_dev,
                                const ScratchLayoutF& L, cudaStream_t st, int dev) {
  constexpr u64 TILE = (u64)NWC * 64 * J;
  constexpr int THREADS = 32 * (NWC + 1 + LBW);
  const u64 full_tiles = n / TILE, rem = n - full_tiles * TILE;
  auto k = filter_ws2_kernel<NWC, S, PC, LBW, D, J, MB, TK, BLK>;
  const int smem = (int)(S * (TILE + 2) * 8);
  PIP_CUDA(cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
  int per_sm = 0;
  PIP_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k, THREADS, smem));
  if (per_sm < 1) return PIP_ERR_UNSUPPORTED;
  if (per_sm > 8) per_sm = 8;
  u64 g = (u64)per_sm * num_sms(dev);
  if (g > full_tiles) g = full_tiles;
  int grid = (int)g;
  u64* mid = rem ? L.carry : m_dev;
  const u32 stride = lb_stride(num_sms(dev), grid);
  PIP_CUDA(cudaMemsetAsync(L.counter, 0, 60, st));
  PIP_CUDA(cudaMemsetAsync(L.slots, 0, sizeof(TileSlot) * 4 * (size_t)grid * stride, st));
  LookbackCtx c{L.slots, L.abort, (u32)(4 * grid), stride};
  DevPred pp = p;
  u32* ticket = L.counter + 2;  // zeroed with the counters above
  void* args[] = {&a, &pp, &mid, &c, (void*)&full_tiles, &ticket};
  PIP_CUDA(cudaLaunchCooperativeKernel((const void*)k, dim3(grid), dim3(THREADS), args, smem, st));
  if (rem) return launch_filter<true>(a + full_tiles * TILE, rem, p, m_dev, L, st, dev, L.carry, a);
  return PIP_OK;
}

template <int NWC, int S, int LBW, int D, int J = 8, int MB = 1, bool TK = false, bool BLK = false>
static int launch_filter_ws2(u64* a, u64 n, const DevPred& p, u64* m_dev, const ScratchLayoutF& L,
                             cudaStream_t st, int dev) {
  switch (pred_class(p)) {
    case PC_MASK: return launch_filter_ws2_pc<NWC, S, PC_MASK, LBW, D, J, MB, TK, BLK>(a, n, p, m_dev, L, st, dev);
    case PC_MOD: return launch_filter_ws2_pc<NWC, S, PC_MOD, LBW, D, J, MB, TK, BLK>(a, n, p, m_dev, L, st, dev);
    case PC_MODODD: return launch_filter_ws2_pc<NWC, S, PC_MODODD, LBW, D, J, MB, TK, BLK>(a, n, p, m_dev, L, st, dev);
    case PC_MODODD0: return launch_filter_ws2_pc<NWC, S, PC_MODODD0, LBW, D, J, MB, TK, BLK>(a, n, p, m_dev, L, st, dev);
    default: return launch_filter_ws2_pc<NWC, S, PC_GEN, LBW, D, J, MB, TK, BLK>(a, n, p, m_dev, L, st, dev);
  }
}

template <int NWC, int S, bool DYN = false, bool AHEAD = false>
static int launch_filter_ws(u64* a, u64 n, const DevPred& p, u64* m_dev, const ScratchLayoutF& L,
                            cudaStream_t st, int dev) {
  switch (pred_class(p)) {
    case PC_MASK: return launch_filter_ws_pc<NWC, S, PC_MASK, DYN, AHEAD>(a, n, p, m_dev, L, st, dev);
    case PC_MOD: return launch_filter_ws_pc<NWC, S, PC_MOD, DYN, AHEAD>(a, n, p, m_dev, L, st, dev);
    case PC_MODODD: return launch_filter_ws_pc<NWC, S, PC_MODODD, DYN, AHEAD>(a, n, p, m_dev, L, st, dev);
    case PC_MODODD0: return launch_filter_ws_pc<NWC, S, PC_MODODD0, DYN, AHEAD>(a, n, p, m_dev, L, st, dev);
    default: return launch_filter_ws_pc<NWC, S, PC_GEN, DYN, AHEAD>(a, n, p, m_dev, L, st, dev);
  }
}

static int filter_cfg() {
  static int cfg = -1;
  if (cfg < 0) {
    // 17 = filter_ws2_kernel<13 compute warps, 4 stages, 3 look-back warps,
    // compaction 2 tiles behind the count> (best measured: 10.36 ms at 2^32;
    // cfg 8 = filter_ws_kernel<16,3> 12.5 ms; <12,4,3,2> 10.66; <13,4,4,2>
    // 10.39; <16,3,3,1> 11.04); 0 = register path; 4/5 = aggregate-ahead TMA
    // 38 (default since the end of round 2) = 14 compute warps (56 KiB tiles,
    // the largest four stages of fit once each lane's keep bits stay in its
    // registers instead of shared memory), 2 look-back warps: 8.40 ms at
    // 2^32 against 8.82 for 17 (39, the same with tiles by ticket: 8.49)
    const char* e = getenv("PIP_FILTER_CFG");
    cfg = e ? atoi(e) : 38;
  }
  return cfg;
}

int filter_device(u64* a, u64 n, const pip_pred* pred, u64* m_dev, void* scratch,
                  size_t scratch_bytes, cudaStream_t st) {
  const int dev = current_device();
  const int sms = num_sms(dev);
  if (!pred || pred->kind > PIP_PRED_EQ) return PIP_ERR_INVALID_ARG;
  if (pred->kind == PIP_PRED_MOD_EQ && pred->a == 0) return PIP_ERR_INVALID_ARG;
  if (!scratch || scratch_bytes < scratch_bytes_for(sms)) return PIP_ERR_OOM;
  if (n == 0) {
    if (m_dev) PIP_CUDA(cudaMemsetAsync(m_dev, 0, 8, st));
    return PIP_OK;
  }
  DevPred p = make_dev_pred(*pred);
  ScratchLayoutF L = carve_f(scratch, sms);
  const bool vec = ((uintptr_t)a & 15) == 0;
  const int cfg = filter_cfg();
  if (vec && cfg >= 6 && n >= 8 * FILTER_TILE) {
    if (cfg == 6) return launch_filter_ws<8, 4>(a, n, p, m_dev, L, st, dev);
    if (cfg == 7) return launch_filter_ws<8, 3>(a, n, p, m_dev, L, st, dev);
    if (cfg == 9) return launch_filter_ws<16, 3, true>(a, n, p, m_dev, L, st, dev);
    if (cfg == 10) return launch_filter_ws<12, 4, false, true>(a, n, p, m_dev, L, st, dev);
    if (cfg == 17) return launch_filter_ws2<13, 4, 3, 2>(a, n, p, m_dev, L, st, dev);  // default
    if (cfg == 35) return launch_filter_ws2<13, 4, 3, 2, 8, 1, true>(a, n, p, m_dev, L, st, dev);  // 17, tiles by ticket
    if (cfg == 38) return launch_filter_ws2<14, 4, 2, 2>(a, n, p, m_dev, L, st, dev);                 // default: 14 compute warps (56 KiB tiles)
    if (cfg == 40) return launch_filter_ws2<14, 4, 3, 2>(a, n, p, m_dev, L, st, dev);                 // the same with 3 look-back warps
    if (cfg == 41) return launch_filter_ws2<14, 4, 2, 2, 8, 1, false, true>(a, n, p, m_dev, L, st, dev);  // 38 with lane-blocked words (no ballots)
    if (cfg == 39) return launch_filter_ws2<14, 4, 2, 2, 8, 1, true>(a, n, p, m_dev, L, st, dev);  // the same, tiles by ticket
    if (cfg == 36) return launch_filter_ws2<13, 4, 2, 2>(a, n, p, m_dev, L, st, dev);                 // 2 look-back warps
    if (cfg == 37) return launch_filter_ws2<13, 4, 2, 2, 8, 1, true>(a, n, p, m_dev, L, st, dev);  // the same, tiles by ticket
    if (cfg == 18) return launch_filter_ws2<12, 4, 3, 2>(a, n, p, m_dev, L, st, dev);
    // half-size tiles (8 words per lane) with twice the stages, so more tile
    // loads are in flight: 14.3 ms (cfg 19) and 12.4 ms (cfg 20: 4 look-back
    // warps, compaction 3 behind) at 2^32 against 9.0 -- the per-tile
    // pipeline, not the loads in flight, paces the filter
    if (cfg == 19) return launch_filter_ws2<13, 8, 3, 2, 4>(a, n, p, m_dev, L, st, dev);
    if (cfg == 20) return launch_filter_ws2<13, 8, 4, 3, 4>(a, n, p, m_dev, L, st, dev);
    // compaction one tile behind the count (one more load in flight, the
    // look-back gets one tile time): 11.0 ms with 3 or 4 look-back warps
    if (cfg == 23) return launch_filter_ws2<13, 4, 3, 1>(a, n, p, m_dev, L, st, dev);
    if (cfg == 24) return launch_filter_ws2<13, 4, 4, 1>(a, n, p, m_dev, L, st, dev);
    // two CTAs per SM, half-size tiles (two independent tile chains per SM)
    if (cfg == 25) return launch_filter_ws2<12, 4, 3, 2, 4, 2>(a, n, p, m_dev, L, st, dev);
    if (cfg == 26) return launch_filter_ws2<12, 4, 2, 2, 4, 2>(a, n, p, m_dev, L, st, dev);
    if (cfg == 27) return launch_filter_ws2<8, 4, 3, 2, 6, 2>(a, n, p, m_dev, L, st, dev);
    // 3/4-size tiles, one more stage (two tile loads in flight behind the
    // two tiles held for the look-back)
    if (cfg == 28) return launch_filter_ws2<13, 5, 3, 2, 6>(a, n, p, m_dev, L, st, dev);
    if (cfg == 29) return launch_filter_ws2<13, 5, 4, 3, 6>(a, n, p, m_dev, L, st, dev);
    if (cfg == 30) return launch_filter_ws2<16, 4, 3, 2, 6>(a, n, p, m_dev, L, st, dev);

    if (cfg == 11) return launch_filter_ws<14, 4>(a, n, p, m_dev, L, st, dev);
    if (cfg == 12) return launch_filter_ws<12, 4>(a, n, p, m_dev, L, st, dev);
    return launch_filter_ws<16, 3>(a, n, p, m_dev, L, st, dev);
  }
  if (vec && cfg >= 4 && n >= 4 * FILTER_TILE) {
    if (cfg == 4) return launch_filter_ahead<512, 3>(a, n, p, m_dev, L, st, dev);
    return launch_filter_ahead<256, 3>(a, n, p, m_dev, L, st, dev);
  }
  if (vec && cfg > 0 && cfg < 4 && n >= FILTER_TILE) {
    if (cfg == 1) return launch_filter_tma<512, 3>(a, n, p, m_dev, L, st, dev);
    if (cfg == 2) return launch_filter_tma<256, 3>(a, n, p, m_dev, L, st, dev);
    return launch_filter_tma<256, 4>(a, n, p, m_dev, L, st, dev);
  }
  return vec ? launch_filter<true>(a, n, p, m_dev, L, st, dev)
             : launch_filter<false>(a, n, p, m_dev, L, st, dev);
}

// memmove inside one array: a[dst : dst+len) = a[src : src+len) (old
// contents).  A left move runs the look-back filter with an always-true
// predicate reading a[src:] and writing from a[dst:] — every tile writes only
// below its own reads, after every earlier tile has read (the in-place
// filter's argument), so overlapping ranges are safe in one pass; disjoint
// ranges are a plain copy; an overlapping right move is a rotation of
// a[src : dst+len) (in place, two passes).
int rotate_device(u64* a, u64 n, u64 o, cudaStream_t st);
int move_device(u64* a, u64 dst, u64 src, u64 len, void* scratch, size_t scratch_bytes,
                cudaStream_t st) {
  const int dev = current_device();
  const int sms = num_sms(dev);
  if (len == 0 || dst == src) return PIP_OK;
  if (!a) return PIP_ERR_INVALID_ARG;
  if (dst + len <= src || src + len <= dst) {
    PIP_CUDA(cudaMemcpyAsync(a + dst, a + src, len * 8, cudaMemcpyDeviceToDevice, st));
    return PIP_OK;
  }
  if (dst > src) return rotate_device(a + src, dst + len - src, len, st);
  if (!scratch || scratch_bytes < scratch_bytes_for(sms)) return PIP_ERR_OOM;
  ScratchLayoutF L = carve_f(scratch, sms);
  const pip_pred all{PIP_PRED_MASK_EQ, 0, 0, 0};
  const DevPred p = make_dev_pred(all);
  u64* from = a + src;
  if (((uintptr_t)from & 15) == 0) return launch_filter<true>(from, len, p, nullptr, L, st, dev, nullptr, a + dst);
  return launch_filter<false>(from, len, p, nullptr, L, st, dev, nullptr, a + dst);
}

int compact_mask_device(u64* a, u64 n, const unsigned char* mask, u64* m_dev, void* scratch,
                        size_t scratch_bytes, cudaStream_t st) {
  const int dev = current_device();
  const int sms = num_sms(dev);
  if ((n && (!a || !mask)) || !m_dev) return PIP_ERR_INVALID_ARG;
  if (!scratch || scratch_bytes < scratch_bytes_for(sms)) return PIP_ERR_OOM;
  if (n == 0) {
    PIP_CUDA(cudaMemsetAsync(m_dev, 0, 8, st));
    return PIP_OK;
  }
  ScratchLayoutF L = carve_f(scratch, sms);
  // the vector path needs 16-byte aligned words and 2-byte aligned flags
  const bool vec = ((uintptr_t)a & 15) == 0 && ((uintptr_t)mask & 1) == 0;
  const u64 tiles = (n + FILTER_TILE - 1) / FILTER_TILE;
  const void* k = vec ? (const void*)compact_mask_kernel<true> : (const void*)compact_mask_kernel<false>;
  int per_sm = 0;
  PIP_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k, FILTER_THREADS, 0));
  if (per_sm < 1) return PIP_ERR_UNSUPPORTED;
  if (per_sm > 8) per_sm = 8;
  u64 g = (u64)per_sm * sms;
  if (g > tiles) g = tiles;
  int grid = (int)g;
  const u32 stride = lb_stride(sms, grid);
  PIP_CUDA(cudaMemsetAsync(L.counter, 0, 60, st));
  PIP_CUDA(cudaMemsetAsync(L.slots, 0, sizeof(TileSlot) * 4 * (size_t)grid * stride, st));
  LookbackCtx c{L.slots, L.abort, (u32)(4 * grid), stride};
  void* args[] = {&a, &n, (void*)&mask, &m_dev, &c, (void*)&tiles};
  PIP_CUDA(cudaLaunchCooperativeKernel(k, dim3(grid), dim3(FILTER_THREADS), args, 0, st));
  return PIP_OK;
}

int count_device(const u64* a, u64 n, const pip_pred* pred, u64* m_dev, void* scratch,
                 size_t scratch_bytes, cudaStream_t st) {
  const int dev = current_device();
  const int sms = num_sms(dev);
  if (!pred || pred->kind > PIP_PRED_EQ || !m_dev) return PIP_ERR_INVALID_ARG;
  if (pred->kind == PIP_PRED_MOD_EQ && pred->a == 0) return PIP_ERR_INVALID_ARG;
  if (!scratch || scratch_bytes < scratch_bytes_for(sms)) return PIP_ERR_OOM;
  DevPred p = make_dev_pred(*pred);
  ScratchLayoutF L = carve_f(scratch, sms);
  int grid = sms * 2;
  u64 need = (n + 1023) / 1024;
  if ((u64)grid > need) grid = (int)(need ? need : 1);
  PIP_CUDA(cudaMemsetAsync(L.counter, 0, 60, st));
  switch (pred_class(p)) {
    case PC_MASK: count_kernel<PC_MASK><<<grid, 512, 0, st>>>(a, n, p, L.partials, L.counter, m_dev); break;
    case PC_MOD: count_kernel<PC_MOD><<<grid, 512, 0, st>>>(a, n, p, L.partials, L.counter, m_dev); break;
    case PC_MODODD: count_kernel<PC_MODODD><<<grid, 512, 0, st>>>(a, n, p, L.partials, L.counter, m_dev); break;
    case PC_MODODD0: count_kernel<PC_MODODD0><<<grid, 512, 0, st>>>(a, n, p, L.partials, L.counter, m_dev); break;
    default: count_kernel<PC_GEN><<<grid, 512, 0, st>>>(a, n, p, L.partials, L.counter, m_dev); break;
  }
  PIP_CHECK_LAUNCH();
  return PIP_OK;
}

// u64 division by an invariant divisor (Granlund-Montgomery / libdivide
// "round-up" method): q = mulhi(x, m) [>> s], with a 65-bit "add" variant.
DevPred make_dev_pred(const pip_pred& in) {
  DevPred p{};
  p.kind = in.kind;
  p.negate = in.negate;
  p.a = in.a;
  p.b = in.b;
  if (in.kind == PIP_PRED_MOD_EQ && in.a >= 1) {
    if (in.b >= in.a) {  // x % d == r with r >= d never holds
      p.kind = PIP_PRED_MASK_EQ;
      p.a = 0;
      p.b = 1;
      return p;
    }
    u64 d = in.a;
    p.tz = (u32)__builtin_ctzll(d);
    const u64 dodd = d >> p.tz;
    u64 inv = dodd;  // Newton: inv <- inv * (2 - d * inv), 6 steps >= 64 bits
    for (int i = 0; i < 6; ++i) inv *= 2 - dodd * inv;
    p.inv = inv;
    p.lim = ~0ull / dodd;
  }
  if (in.kind == PIP_PRED_MOD_EQ && in.a >= 1) {
    const u64 d = in.a;
    if ((d & (d - 1)) == 0) {
      p.pow2 = 1;
    } else {
      int l = 63 - __builtin_clzll(d);  // floor(log2 d); d not a power of 2
      unsigned __int128 one = 1;
      // m = floor(2^(64+l) / d) + 1 ; check if it fits 64 bits with error bound
      unsigned __int128 num = one << (64 + l);
      u64 proposed = (u64)(num / d);
      u64 rem = (u64)(num - (unsigned __int128)proposed * d);
      u64 e = d - rem;
      if (e < (1ull << l)) {
        p.magic = proposed + 1;
        p.shift = l;
        p.add = 0;
      } else {
        // 65-bit multiplier: m = 2*proposed + 1 (mod 2^64), add-indicator form
        proposed += proposed;
        u64 twice_rem = rem + rem;
        if (twice_rem >= d || twice_rem < rem) proposed += 1;
        p.magic = proposed + 1;
        p.shift = l;
        p.add = 1;
      }
    }
  }
  return p;
}

}  // namespace pip
