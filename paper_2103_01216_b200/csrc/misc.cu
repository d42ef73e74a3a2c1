// Rotation (strong.rotate), swap-sequence validation, input generation
// (runtime.Rng, relaxed.make_swap_sequence) and the random-access
// microbenchmark used as the permutation's roofline denominator.
#include "common.cuh"

namespace pip {

// ---------------------------------------------------------------------------
// rotate: strong.py:67-95 (triple reversal, 256-word swaps per step).
// Same triple reversal, each reversal one coalesced kernel: thread k swaps
// a[s+k] <-> a[t-1-k] for k < (t-s)/2 (both sides contiguous runs).
__global__ void reverse_kernel(u64* __restrict__ a, u64 s, u64 t) {
  const u64 half = (t - s) / 2;
  const u64 stride = (u64)gridDim.x * blockDim.x;
  for (u64 k = (u64)blockIdx.x * blockDim.x + threadIdx.x; k < half; k += stride) {
    u64* l = a + s + k;
    u64* r = a + t - 1 - k;
    u64 x = *l, y = *r;
    *l = y;
    *r = x;
  }
}

static int reverse(u64* a, u64 s, u64 t, cudaStream_t st) {
  if (t - s < 2) return PIP_OK;
  const u64 half = (t - s) / 2;
  u64 blocks = (half + 255) / 256;
  const u64 cap = (u64)num_sms(current_device()) * 16;
  if (blocks > cap) blocks = cap;
  reverse_kernel<<<(unsigned)blocks, 256, 0, st>>>(a, s, t);
  PIP_CHECK_LAUNCH();
  return PIP_OK;
}

int reverse_device(u64* a, u64 n, cudaStream_t st) { return reverse(a, 0, n, st); }

int rotate_device(u64* a, u64 n, u64 o, cudaStream_t st) {
  if (o > n) return PIP_ERR_INVALID_ARG;
  if (o == 0 || o == n || n < 2) return PIP_OK;
  int rc;
  if ((rc = reverse(a, 0, o, st))) return rc;
  if ((rc = reverse(a, o, n, st))) return rc;
  return reverse(a, 0, n, st);
}

// ---------------------------------------------------------------------------
// validate_swap_sequence (relaxed.py:55-58) fused with the non-self count
// (relaxed.py:239).  counters[0] = #nonself, counters[1] = #invalid.
__global__ void validate_kernel(const u64* __restrict__ h, u64 n, u64* counters) {
  u64 ns = 0, bad = 0;
  const u64 stride = (u64)gridDim.x * blockDim.x;
  for (u64 i = (u64)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride) {
    const u64 v = h[i];
    ns += v != i;
    bad += v > i;
  }
  ns = warp_reduce<Op<PIP_OP_ADD>>(ns);
  bad = warp_reduce<Op<PIP_OP_ADD>>(bad);
  if (lane_id() == 0) {
    if (ns) atomicAdd(counters, ns);
    if (bad) atomicAdd(counters + 1, bad);
  }
}

// the same pass, also writing the non-self count of every 4096-id block
// (bcnt[c] for ids [4096c, 4096c + 4096)): the permutation's window counts
// then come from these instead of a second read of H
static constexpr u32 VBLK_SHIFT = 12;
__global__ void __launch_bounds__(256) validate_blocks_kernel(const u64* __restrict__ h, u64 n,
                                                              u64* counters, u32* bcnt) {
  __shared__ u32 s_w[8];
  const u64 nblk = (n + (1ull << VBLK_SHIFT) - 1) >> VBLK_SHIFT;
  u64 ns_all = 0, bad_all = 0;
  for (u64 c = blockIdx.x; c < nblk; c += gridDim.x) {
    const u64 base = c << VBLK_SHIFT;
    u32 ns = 0;
#pragma unroll 4
    for (u32 q = threadIdx.x; q < (1u << VBLK_SHIFT); q += 256) {
      const u64 i = base + q;
      if (i < n) {
        const u64 v = __ldcs(h + i);
        ns += v != i;
        bad_all += v > i;
      }
    }
    ns = __reduce_add_sync(0xffffffffu, ns);
    if (lane_id() == 0) s_w[warp_id()] = ns;
    __syncthreads();
    if (threadIdx.x == 0) {
      u32 t = 0;
      for (int w = 0; w < 8; ++w) t += s_w[w];
      bcnt[c] = t;
      ns_all += t;
    }
    __syncthreads();
  }
  bad_all = warp_reduce<Op<PIP_OP_ADD>>(bad_all);
  if (lane_id() == 0 && bad_all) atomicAdd(counters + 1, bad_all);
  if (threadIdx.x == 0 && ns_all) atomicAdd(counters, ns_all);
}

int validate_counts(const u64* h, u64 n, u64* nonself, u64* invalid, void* scratch16,
                    cudaStream_t st, u32* bcnt) {
  u64* cnt = (u64*)scratch16;
  PIP_CUDA(cudaMemsetAsync(cnt, 0, 16, st));
  if (n && bcnt) {
    const u64 nblk = (n + (1ull << VBLK_SHIFT) - 1) >> VBLK_SHIFT;
    u64 blocks = nblk;
    const u64 cap = (u64)num_sms(current_device()) * 8;
    if (blocks > cap) blocks = cap;
    validate_blocks_kernel<<<(unsigned)blocks, 256, 0, st>>>(h, n, cnt, bcnt);
    PIP_CHECK_LAUNCH();
  } else if (n) {
    u64 blocks = (n + 255) / 256;
    const u64 cap = (u64)num_sms(current_device()) * 8;
    if (blocks > cap) blocks = cap;
    validate_kernel<<<(unsigned)blocks, 256, 0, st>>>(h, n, cnt);
    PIP_CHECK_LAUNCH();
  }
  if (!nonself) return PIP_OK;  // stream-ordered: the caller reads cnt[0..1] on the device
  u64 host[2];
  PIP_CUDA(cudaMemcpyAsync(host, cnt, 16, cudaMemcpyDeviceToHost, st));
  PIP_CUDA(cudaStreamSynchronize(st));
  *nonself = host[0];
  *invalid = host[1];
  return PIP_OK;
}

int validate_device(const u64* h, u64 n, u64* nonself_dev, void* scratch, size_t scratch_bytes,
                    cudaStream_t st) {
  if (!scratch || scratch_bytes < 16) return PIP_ERR_OOM;
  u64 ns = 0, bad = 0;
  int rc = validate_counts(h, n, &ns, &bad, scratch, st, nullptr);
  if (rc) return rc;
  if (nonself_dev) {
    PIP_CUDA(cudaMemcpyAsync(nonself_dev, &ns, 8, cudaMemcpyHostToDevice, st));
    PIP_CUDA(cudaStreamSynchronize(st));
  }
  return bad ? PIP_ERR_INVALID_SWAPS : PIP_OK;
}

// ---------------------------------------------------------------------------
// Rng.words / make_swap_sequence (runtime.py:293-295, relaxed.py:47-52)
__global__ void rng_words_kernel(u64* __restrict__ out, u64 lo, u64 count, u64 seed, u32 shift) {
  const u64 stride = (u64)gridDim.x * blockDim.x;
  for (u64 k = (u64)blockIdx.x * blockDim.x + threadIdx.x; k < count; k += stride)
    out[k] = mix64((lo + k + 1) * GOLDEN + seed) >> shift;
}
__global__ void make_swaps_kernel(u64* __restrict__ out, u64 lo, u64 count, u64 seed) {
  const u64 stride = (u64)gridDim.x * blockDim.x;
  for (u64 k = (u64)blockIdx.x * blockDim.x + threadIdx.x; k < count; k += stride) {
    const u64 i = lo + k;
    out[k] = mix64((i + 1) * GOLDEN + seed) % (i + 1);
  }
}

int rng_words(u64* out, u64 lo, u64 count, u64 seed, u32 shift, cudaStream_t st) {
  if (shift > 63) return PIP_ERR_INVALID_ARG;
  if (!count) return PIP_OK;
  u64 blocks = (count + 255) / 256;
  const u64 cap = (u64)num_sms(current_device()) * 16;
  if (blocks > cap) blocks = cap;
  rng_words_kernel<<<(unsigned)blocks, 256, 0, st>>>(out, lo, count, seed, shift);
  PIP_CHECK_LAUNCH();
  return PIP_OK;
}
int make_swaps(u64* out, u64 lo, u64 count, u64 seed, cudaStream_t st) {
  if (!count) return PIP_OK;
  u64 blocks = (count + 255) / 256;
  const u64 cap = (u64)num_sms(current_device()) * 16;
  if (blocks > cap) blocks = cap;
  make_swaps_kernel<<<(unsigned)blocks, 256, 0, st>>>(out, lo, count, seed);
  PIP_CHECK_LAUNCH();
  return PIP_OK;
}

// ---------------------------------------------------------------------------
// random 8-byte read-modify-write microbenchmark (the RP roofline: the swap
// phase touches 2 random 32-byte sectors per committed swap)
template <int MODE>
__global__ void __launch_bounds__(256)
random_rmw_kernel(u64* __restrict__ buf, u64 n, u64 updates, u64 seed) {
  // 8 independent read-modify-writes in flight per thread; index by
  // multiply-high range reduction (no 64-bit division on the critical path).
  // MODE 0: load + store (two requests per update); 1: one atomic exchange
  // whose old value is consumed (the swap's form); 2: a reduction (no
  // return value)
  const u64 stride = (u64)gridDim.x * blockDim.x;
  u64 acc = 0;
  for (u64 k = (u64)blockIdx.x * blockDim.x + threadIdx.x; k * 8 < updates; k += stride) {
    u64 idx[8], v[8];
#pragma unroll
    for (int q = 0; q < 8; ++q) idx[q] = __umul64hi(mix64(seed + (k * 8 + q) * GOLDEN), n);
    if (MODE == 0) {
#pragma unroll
      for (int q = 0; q < 8; ++q) v[q] = __ldcg(buf + idx[q]);
#pragma unroll
      for (int q = 0; q < 8; ++q) buf[idx[q]] = v[q] + 1;
    } else if (MODE == 1) {
#pragma unroll
      for (int q = 0; q < 8; ++q) v[q] = atomicExch((unsigned long long*)buf + idx[q], (unsigned long long)(k + q));
#pragma unroll
      for (int q = 0; q < 8; ++q) acc += v[q];
    } else {
#pragma unroll
      for (int q = 0; q < 8; ++q) atomicAdd((unsigned long long*)buf + idx[q], 1ull);
    }
  }
  if (MODE == 1 && acc == 0x123456789abcdefull) buf[0] = acc;  // keep the exchanges' results live
}

int bench_random_rmw(u64* buf, u64 n, u64 updates, u64 seed, float* ms, cudaStream_t st, int mode) {
  if (!n || mode > 2) return PIP_ERR_INVALID_ARG;
  cudaEvent_t e0, e1;
  PIP_CUDA(cudaEventCreate(&e0));
  PIP_CUDA(cudaEventCreate(&e1));
  const int blocks = num_sms(current_device()) * 8;
  // mode: 0 load + store, 1 atomic exchange (the form the scheme-3 swaps
  // use), 2 reduction; < 0: PIP_RMW_MODE (measurement knob), default 0
  if (mode < 0) mode = getenv("PIP_RMW_MODE") ? atoi(getenv("PIP_RMW_MODE")) : 0;
  auto kern = mode == 1 ? random_rmw_kernel<1> : mode == 2 ? random_rmw_kernel<2> : random_rmw_kernel<0>;
  kern<<<blocks, 256, 0, st>>>(buf, n, updates / 8, seed ^ 0x5555);  // warm
  PIP_CUDA(cudaEventRecord(e0, st));
  kern<<<blocks, 256, 0, st>>>(buf, n, updates, seed);
  PIP_CUDA(cudaEventRecord(e1, st));
  PIP_CUDA(cudaEventSynchronize(e1));
  PIP_CUDA(cudaEventElapsedTime(ms, e0, e1));
  cudaEventDestroy(e0);
  cudaEventDestroy(e1);
  return PIP_OK;
}

}  // namespace pip
