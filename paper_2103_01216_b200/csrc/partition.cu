// Unstable in-place partition (strong.partition_unstable, strong.py:394-419;
// relaxed.partition_relaxed, relaxed.py:312-344): on return the words with
// pred true occupy a[0:m), the others a[m:n), the multiset is preserved and
// m = #true is returned.  The reference's order inside each side is
// unspecified ("unstable"; its tests check exactly this contract,
// test_strong.py:189-207), so any placement that meets it is a drop-in.
//
// B200 design — in place, swap-based, O(n/T) device descriptors (T = 4096):
//   K1 count   per-tile true counts tc[k] (8 B/word, streaming).
//   K2 plan    (one CTA) m = sum tc and the boundary tile's true count left
//              of m; misfits are the false words left of m and the true words
//              right of m (equally many, X); exclusive prefix sums of the
//              per-tile misfit counts give ranks: left misfit of rank r is
//              exchanged with right misfit of rank r.
//   K3 bounds  (read-only) for every left tile with misfits, the position of
//              the right misfit whose rank is the tile's first rank (binary
//              search over the right tiles' rank bases, then a warp ballot
//              scan of that tile) -> startR[k].  The right misfits of tile k
//              are the first cnt_k true words at positions >= startR[k];
//              the positions in between are untouched false words.
//   K4 swap    one CTA per left tile: its misfits and its cnt_k right
//              misfits are collected (positions + values) in shared memory
//              and exchanged.  Every position a CTA reads or writes is
//              exclusive to it, so the predicate values it reads are the
//              original ones and no CTA waits for another.
// Traffic: 8 B/word (count) + ~8 B/word (swap reads) + the misfits' writes
// + half a tile per left tile for the bounds (K3).
#include <cstdio>
#include "sync.cuh"

namespace pip {

static constexpr u32 PT_LOG = 12;
static constexpr u64 PT = 1ull << PT_LOG;  // words per tile
static constexpr int PT_THREADS = 256;
static constexpr int PT_PER = (int)(PT / PT_THREADS);  // 16 words per thread

struct PartInfo {
  u64 m, X, kb, nleft;  // #true, #misfit pairs, boundary tile, tiles with a left part
};

// ---------------------------------------------------------------- K1 count
__global__ void __launch_bounds__(PT_THREADS) part_count_kernel(const u64* __restrict__ a, u64 n,
                                                                DevPred p, u32* __restrict__ tc,
                                                                u64 ntiles) {
  __shared__ u32 s_w[PT_THREADS / 32];
  for (u64 k = blockIdx.x; k < ntiles; k += gridDim.x) {
    const u64 base = k * PT;
    u32 c = 0;
#pragma unroll
    for (int q = 0; q < PT_PER; ++q) {
      const u64 i = base + threadIdx.x + (u64)q * PT_THREADS;
      if (i < n) c += (u32)pred_eval(p, __ldcs(a + i));
    }
    c = __reduce_add_sync(0xffffffffu, c);
    if ((threadIdx.x & 31) == 0) s_w[threadIdx.x >> 5] = c;
    __syncthreads();
    if (threadIdx.x == 0) {
      u32 t = 0;
      for (int w = 0; w < PT_THREADS / 32; ++w) t += s_w[w];
      tc[k] = t;
    }
    __syncthreads();
  }
}

// ---------------------------------------------------------------- K2 plan
// one CTA of 1024 threads; each thread owns a contiguous run of tiles
static constexpr int PL_THREADS = 1024;

__device__ __forceinline__ void tile_mis(u64 k, u64 n, u64 m, u64 kb, u32 tl, const u32* tc,
                                         u64& ml, u64& mr) {
  const u64 lo = k * PT, hi = lo + PT < n ? lo + PT : n;
  const u64 ll = m <= lo ? 0 : (m >= hi ? hi - lo : m - lo);  // words left of m
  const u64 tleft = k < kb ? tc[k] : (k == kb ? tl : 0);        // true words left of m
  ml = ll - tleft;
  mr = tc[k] - tleft;
}

__global__ void __launch_bounds__(PL_THREADS) part_plan_kernel(const u64* __restrict__ a, u64 n,
                                                               DevPred p, const u32* __restrict__ tc,
                                                               u64 ntiles, u64* baseL, u64* baseR,
                                                               PartInfo* info, u64* m_dev) {
  __shared__ u64 s_a[PL_THREADS], s_b[PL_THREADS];
  __shared__ u64 s_m;
  __shared__ u32 s_tl;
  const u32 t = threadIdx.x;
  const u64 per = (ntiles + PL_THREADS - 1) / PL_THREADS;
  const u64 k0 = t * per < ntiles ? t * per : ntiles, k1 = k0 + per < ntiles ? k0 + per : ntiles;
  // m
  u64 s = 0;
  for (u64 k = k0; k < k1; ++k) s += tc[k];
  s_a[t] = s;
  if (t == 0) s_tl = 0;
  __syncthreads();
  for (u32 o = PL_THREADS / 2; o > 0; o >>= 1) {
    if (t < o) s_a[t] += s_a[t + o];
    __syncthreads();
  }
  if (t == 0) s_m = s_a[0];
  __syncthreads();
  const u64 m = s_m;
  const u64 kb = m / PT;  // tile holding position m (== ntiles if m == n and n % PT == 0)
  // true words of tile kb left of m
  if (kb < ntiles) {
    u32 c = 0;
    for (u64 i = kb * PT + t; i < m; i += PL_THREADS) c += (u32)pred_eval(p, a[i]);
    c = __reduce_add_sync(0xffffffffu, c);
    if ((t & 31) == 0 && c) atomicAdd(&s_tl, c);
  }
  __syncthreads();
  const u32 tl = s_tl;
  // exclusive scans of the per-tile misfit counts
  u64 sl = 0, sr = 0;
  for (u64 k = k0; k < k1; ++k) {
    u64 ml, mr;
    tile_mis(k, n, m, kb, tl, tc, ml, mr);
    sl += ml;
    sr += mr;
  }
  __syncthreads();
  s_a[t] = sl;
  s_b[t] = sr;
  __syncthreads();
  for (u32 o = 1; o < PL_THREADS; o <<= 1) {  // Hillis-Steele inclusive scan
    const u64 xa = t >= o ? s_a[t - o] : 0, xb = t >= o ? s_b[t - o] : 0;
    __syncthreads();
    s_a[t] += xa;
    s_b[t] += xb;
    __syncthreads();
  }
  u64 el = s_a[t] - sl, er = s_b[t] - sr;
  for (u64 k = k0; k < k1; ++k) {
    u64 ml, mr;
    tile_mis(k, n, m, kb, tl, tc, ml, mr);
    baseL[k] = el;
    baseR[k] = er;
    el += ml;
    er += mr;
  }
  if (t == PL_THREADS - 1) {
    info->m = m;
    info->X = s_a[t];  // == s_b[t]
    info->kb = kb;
    info->nleft = (m + PT - 1) / PT;
    *m_dev = m;
  }
}

// ---------------------------------------------------------------- K3 bounds
// one warp per left tile k with misfits: position of right misfit rank baseL[k]
__global__ void __launch_bounds__(256) part_bounds_kernel(const u64* __restrict__ a, u64 n, DevPred p,
                                                          const u32* __restrict__ tc,
                                                          const u64* __restrict__ baseL,
                                                          const u64* __restrict__ baseR, u64 ntiles,
                                                          const PartInfo* info, u64* startR) {
  const u64 m = info->m, X = info->X, nleft = info->nleft, kb = info->kb;
  if (X == 0) return;
  const u32 lane = threadIdx.x & 31;
  const u64 nw = (u64)gridDim.x * (blockDim.x >> 5);
  for (u64 k = (u64)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5); k < nleft; k += nw) {
    const u64 r = baseL[k];
    const u64 rn = k + 1 < ntiles ? baseL[k + 1] : X;
    if (rn <= r) continue;  // no misfits in this left tile
    // right tile j: largest j in [kb, ntiles) with baseR[j] <= r
    u64 lo = kb, hi = ntiles;  // invariant: baseR[lo] <= r (baseR[kb] == 0)
    while (hi - lo > 1) {
      const u64 mid = (lo + hi) >> 1;
      if (baseR[mid] <= r) lo = mid;
      else hi = mid;
    }
    const u64 j = lo;
    u64 q = r - baseR[j];  // rank inside tile j
    const u64 s0 = j * PT > m ? j * PT : m, s1 = (j + 1) * PT < n ? (j + 1) * PT : n;
    u64 pos = ~0ull;
    for (u64 i0 = s0; i0 < s1; i0 += 32) {
      const u64 i = i0 + lane;
      const bool f = i < s1 && pred_eval(p, a[i]);
      const unsigned bal = __ballot_sync(0xffffffffu, f);
      const u32 c = __popc(bal);
      if (q < c) {
        // the (q+1)-th set bit of bal
        unsigned b = bal;
        for (u64 z = 0; z < q; ++z) b &= b - 1;
        pos = i0 + (u64)(__ffs(b) - 1);
        break;
      }
      q -= c;
    }
    if (lane == 0) startR[k] = pos;
  }
  (void)tc;
}

// ---------------------------------------------------------------- K4 swap
struct PartSmem {
  u64 lval[PT];
  u64 rval[PT];
  u32 rpos[PT];  // offset from startR[k]
  unsigned short lpos[PT];
  u32 cnt_l, cnt_r;
  u32 warp[PT_THREADS / 32];
};

__global__ void __launch_bounds__(PT_THREADS) part_swap_kernel(u64* a, u64 n, DevPred p,
                                                               const u64* __restrict__ baseL, u64 ntiles,
                                                               const PartInfo* info,
                                                               const u64* __restrict__ startR) {
  extern __shared__ __align__(16) unsigned char smraw[];
  PartSmem& S = *reinterpret_cast<PartSmem*>(smraw);
  const u64 m = info->m, X = info->X, nleft = info->nleft;
  if (X == 0) return;
  const u32 tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
  for (u64 k = blockIdx.x; k < nleft; k += gridDim.x) {
    const u64 r = baseL[k];
    const u64 rn = k + 1 < ntiles ? baseL[k + 1] : X;
    if (rn <= r) continue;
    const u32 cnt = (u32)(rn - r);
    // left misfits: false words of [kT, min((k+1)T, m))
    if (tid == 0) { S.cnt_l = 0; S.cnt_r = 0; }
    __syncthreads();
    const u64 lo = k * PT, hi = lo + PT < m ? lo + PT : m;
#pragma unroll
    for (int q = 0; q < PT_PER; ++q) {
      const u64 i = lo + tid + (u64)q * PT_THREADS;
      if (i < hi) {
        const u64 v = a[i];
        if (!pred_eval(p, v)) {
          const u32 s = atomicAdd(&S.cnt_l, 1u);
          S.lval[s] = v;
          S.lpos[s] = (unsigned short)(i - lo);
        }
      }
    }
    // right misfits: the first cnt true words at positions >= startR[k]
    const u64 sr = startR[k];
    u32 got = 0;  // uniform
    for (u64 i0 = sr; got < cnt && i0 < n; i0 += PT_THREADS * 4) {
      u64 v[4];
      bool f[4];
      u32 c = 0;
#pragma unroll
      for (int q = 0; q < 4; ++q) {  // thread-contiguous: position order = (tid, q)
        const u64 i = i0 + (u64)tid * 4 + q;
        v[q] = i < n ? a[i] : 0ull;
        f[q] = i < n && pred_eval(p, v[q]);
        c += f[q];
      }
      // block exclusive scan of c
      u32 x = c;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const u32 y = __shfl_up_sync(0xffffffffu, x, o);
        if (lane >= (u32)o) x += y;
      }
      if (lane == 31) S.warp[wid] = x;
      __syncthreads();
      u32 wbase = 0, tot = 0;
      for (int w = 0; w < PT_THREADS / 32; ++w) {
        const u32 ww = S.warp[w];
        wbase += (u32)w < wid ? ww : 0u;
        tot += ww;
      }
      u32 rank = got + wbase + x - c;
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        if (f[q] && rank < cnt) {
          S.rval[rank] = v[q];
          S.rpos[rank] = (u32)(i0 + (u64)tid * 4 + q - sr);
        }
        rank += f[q];
      }
      got += tot;
      __syncthreads();
    }
    __syncthreads();
    // exchange (cnt_l == cnt by construction)
    for (u32 s = tid; s < cnt; s += PT_THREADS) {
      a[lo + S.lpos[s]] = S.rval[s];
      a[sr + S.rpos[s]] = S.lval[s];
    }
    __syncthreads();
  }
}

// ---------------------------------------------------------------- host
struct PartLayout {
  size_t tc, baseL, baseR, startR, info, total;
};

static PartLayout part_layout(u64 n) {
  const u64 ntiles = (n + PT - 1) / PT;
  PartLayout L{};
  size_t off = 0;
  auto take = [&](size_t bytes) {
    size_t o = off;
    off += (bytes + 255) & ~(size_t)255;
    return o;
  };
  L.tc = take(ntiles * 4);
  L.baseL = take(ntiles * 8);
  L.baseR = take(ntiles * 8);
  L.startR = take(ntiles * 8);
  L.info = take(sizeof(PartInfo));
  L.total = off;
  return L;
}

size_t partition_workspace_bytes(u64 n) { return n ? part_layout(n).total : 0; }

int partition_device(u64* a, u64 n, const pip_pred* pred, u64* m_dev, void* ws, size_t ws_bytes,
                     cudaStream_t st) {
  if (!pred || !m_dev) return PIP_ERR_INVALID_ARG;
  if (n == 0) {
    PIP_CUDA(cudaMemsetAsync(m_dev, 0, 8, st));
    return PIP_OK;
  }
  if (n > (1ull << 32)) return PIP_ERR_UNSUPPORTED;  // u32 right offsets in K4
  const PartLayout L = part_layout(n);
  if (!ws || ws_bytes < L.total) return PIP_ERR_OOM;
  char* w = (char*)ws;
  u32* tc = (u32*)(w + L.tc);
  u64* baseL = (u64*)(w + L.baseL);
  u64* baseR = (u64*)(w + L.baseR);
  u64* startR = (u64*)(w + L.startR);
  PartInfo* info = (PartInfo*)(w + L.info);
  const u64 ntiles = (n + PT - 1) / PT;
  const DevPred p = make_dev_pred(*pred);
  const int sms = num_sms(current_device());
  const u64 g1 = ntiles < (u64)sms * 8 ? ntiles : (u64)sms * 8;
  part_count_kernel<<<(unsigned)g1, PT_THREADS, 0, st>>>(a, n, p, tc, ntiles);
  PIP_CHECK_LAUNCH();
  part_plan_kernel<<<1, PL_THREADS, 0, st>>>(a, n, p, tc, ntiles, baseL, baseR, info, m_dev);
  PIP_CHECK_LAUNCH();
  const u64 g3 = (ntiles + 7) / 8 < (u64)sms * 8 ? (ntiles + 7) / 8 : (u64)sms * 8;
  part_bounds_kernel<<<(unsigned)g3, 256, 0, st>>>(a, n, p, tc, baseL, baseR, ntiles, info, startR);
  PIP_CHECK_LAUNCH();
  const size_t smem = sizeof(PartSmem);
  PIP_CUDA(cudaFuncSetAttribute(part_swap_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                (int)smem));
  const u64 g4 = ntiles < (u64)sms * 2 ? ntiles : (u64)sms * 2;
  part_swap_kernel<<<(unsigned)g4, PT_THREADS, smem, st>>>(a, n, p, baseL, ntiles, info, startR);
  PIP_CHECK_LAUNCH();
  return PIP_OK;
}

}  // namespace pip
