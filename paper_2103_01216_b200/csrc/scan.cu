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
#include "lookback.cuh"

namespace pip {

static constexpr int SCAN_THREADS = 512;
static constexpr int SCAN_ITEMS = 16;
static constexpr u64 SCAN_TILE = (u64)SCAN_THREADS * SCAN_ITEMS;  // 8192

template <int OP, bool INCLUSIVE, bool VEC>
__global__ void __launch_bounds__(SCAN_THREADS, 2)
scan_kernel(u64* __restrict__ a, u64 n, u64 init, const u64* carry_in, u64* total, LookbackCtx c,
            u64 num_tiles) {
  using O = Op<OP>;
  __shared__ u64 s_warp[SCAN_THREADS / 32];
  __shared__ int s_abort;
  const u32 lane = lane_id(), warp = warp_id();

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
    // tile aggregate
    u64 t = x[0];
#pragma unroll
    for (int k = 1; k < SCAN_ITEMS; ++k) t = O::apply(t, x[k]);
    t = warp_reduce<O>(t);
    if (lane == 0) s_warp[warp] = t;
    __syncthreads();
    if (warp == 0) {
      u64 wv = lane < SCAN_THREADS / 32 ? s_warp[lane] : O::identity;
      u64 winc = warp_incl_scan<O>(wv);
      u64 wexc = __shfl_up_sync(0xffffffffu, winc, 1);
      if (lane == 0) wexc = O::identity;
      const u64 agg = __shfl_sync(0xffffffffu, winc, SCAN_THREADS / 32 - 1);
      // carry_in (streaming chunks) acts as an inclusive tile -1
      u64 prefix = (tile == 0 && carry_in) ? *carry_in : O::identity;
      int ok = 1;
      if (lane == 0) {
        ok = publish_begin(c, tile);
        if (ok) {
          if (tile == 0) publish_incl(c, tile, O::apply(prefix, agg));
          else publish_agg(c, tile, agg);
        }
      }
      ok = __shfl_sync(0xffffffffu, ok, 0);
      if (ok && tile > 0) {
        ok = lookback<O>(c, tile, prefix);
        if (ok && lane == 0) publish_incl(c, tile, O::apply(prefix, agg));
      }
      if (lane < SCAN_THREADS / 32) s_warp[lane] = O::apply(prefix, wexc);
      if (lane == 0) {
        s_abort = !ok;
        if (ok && tile == num_tiles - 1 && total) *total = O::apply(prefix, agg);
      }
    }
    __syncthreads();
    if (s_abort) return;
    u64 run = s_warp[warp];
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
  u64* partials;    // G_MAX
  TileSlot* slots;  // 2 * G_MAX
};
static constexpr int CTAS_PER_SM_MAX = 8;
static size_t header_bytes() { return 256; }
size_t scratch_bytes_for(int sms) {
  const size_t gmax = (size_t)sms * CTAS_PER_SM_MAX;
  return header_bytes() + gmax * sizeof(u64) + 2 * gmax * sizeof(TileSlot);
}
static ScratchLayout carve(void* scratch, int sms) {
  const size_t gmax = (size_t)sms * CTAS_PER_SM_MAX;
  char* p = (char*)scratch;
  ScratchLayout L;
  L.abort = (u32*)p;
  L.counter = (u32*)p + 1;
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
  PIP_CUDA(cudaMemsetAsync(L.abort, 0, header_bytes(), st));
  PIP_CUDA(cudaMemsetAsync(L.slots, 0, sizeof(TileSlot) * 2 * (size_t)grid, st));
  LookbackCtx c{L.slots, L.abort, (u32)grid};
  void* args[] = {&a, &n, &init, &carry, &total, &c, (void*)&tiles};
  PIP_CUDA(cudaLaunchCooperativeKernel((const void*)k, dim3(grid), dim3(SCAN_THREADS), args, 0, st));
  return PIP_OK;
}

template <int OP>
static int launch_scan_op(u64* a, u64 n, u64 init, int inclusive, const u64* carry, u64* total,
                          const ScratchLayout& L, cudaStream_t st, int device) {
  const bool vec = ((uintptr_t)a & 15) == 0;
  if (inclusive) {
    return vec ? launch_scan_t<OP, true, true>(a, n, init, carry, total, L, st, device)
               : launch_scan_t<OP, true, false>(a, n, init, carry, total, L, st, device);
  }
  return vec ? launch_scan_t<OP, false, true>(a, n, init, carry, total, L, st, device)
             : launch_scan_t<OP, false, false>(a, n, init, carry, total, L, st, device);
}

int check_abort(void* scratch, cudaStream_t st) {
  u32 h = 0;
  PIP_CUDA(cudaMemcpyAsync(&h, scratch, sizeof(u32), cudaMemcpyDeviceToHost, st));
  PIP_CUDA(cudaStreamSynchronize(st));
  return h ? PIP_ERR_CUDA : PIP_OK;
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
  PIP_CUDA(cudaMemsetAsync(L.abort, 0, header_bytes(), st));
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
