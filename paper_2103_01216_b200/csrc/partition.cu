// Unstable in-place partition (strong.partition_unstable, strong.py:394-419;
// relaxed.partition_relaxed, relaxed.py:312-344): on return the words with
// pred true occupy a[0:m), the others a[m:n), the multiset is preserved and
// m = #true is returned.  The reference's order inside each side is
// unspecified ("unstable"; its tests check exactly this contract,
// test_strong.py:189-207), so any placement that meets it is a drop-in.
//
// B200 design — in place, swap-based, O(n/T) device descriptors (T = 2048):
//   K1 count   per-tile true counts tc[k] (8 B/word, streaming).
//   K2 plan    (group sums, one CTA, group rescans) m = sum tc and the
//              boundary tile's true count left
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

static constexpr u32 PT_LOG = 11;
static constexpr u64 PT = 1ull << PT_LOG;  // words per tile
static constexpr int PT_THREADS = 256;
static constexpr int PT_PER = (int)(PT / PT_THREADS);  // 8 words per thread

struct PartInfo {
  u64 m, X, kb, nleft;  // #true, #misfit pairs, boundary tile, tiles with a left part
  u64 tl;               // true words of tile kb left of m
};

static int part_pred_class(const DevPred& p) {
  if (p.kind == PIP_PRED_MASK_EQ) return PC_MASK;
  if (p.kind == PIP_PRED_MOD_EQ) return p.tz == 0 ? (p.b == 0 ? PC_MODODD0 : PC_MODODD) : PC_MOD;
  return PC_GEN;
}

// ---------------------------------------------------------------- K1 count
template <int PC>
__global__ void __launch_bounds__(PT_THREADS) part_count_kernel(const u64* __restrict__ a, u64 n,
                                                                DevPred p, u32* __restrict__ tc,
                                                                u64 ntiles) {
  __shared__ u32 s_w[PT_THREADS / 32];
  for (u64 k = blockIdx.x; k < ntiles; k += gridDim.x) {
    const u64 base = k * PT;
    u64 v[PT_PER];
#pragma unroll
    for (int q = 0; q < PT_PER; ++q) {
      const u64 i = base + threadIdx.x + (u64)q * PT_THREADS;
      v[q] = i < n ? __ldcs(a + i) : 0ull;
    }
    u32 c = 0;
#pragma unroll
    for (int q = 0; q < PT_PER; ++q)
      c += (u32)(base + threadIdx.x + (u64)q * PT_THREADS < n && pred_eval_t<PC>(p, v[q]));
    c = __reduce_add_sync(0xffffffffu, c);
    if ((threadIdx.x & 31) == 0) s_w[threadIdx.x >> 5] = c;
    __syncthreads();
    if (threadIdx.x < 32) {
      u32 t = threadIdx.x < PT_THREADS / 32 ? s_w[threadIdx.x] : 0u;
      t = __reduce_add_sync(0xffffffffu, t);
      if (threadIdx.x == 0) tc[k] = t;
    }
    __syncthreads();
  }
}

// ---------------------------------------------------------------- K2 plan
// three small launches: per-group sums of tc (PL_GROUPS CTAs) -> one CTA: m,
// the boundary tile, the groups' misfit sums and their exclusive scan ->
// per-group rescan writing baseL / baseR (PL_GROUPS CTAs)
static constexpr int PL_THREADS = 1024;
static constexpr int PL_GROUPS = 1024;

__device__ __forceinline__ void tile_mis(u64 k, u64 n, u64 m, u64 kb, u32 tl, u32 tck, u64& ml,
                                         u64& mr) {
  const u64 lo = k * PT, hi = lo + PT < n ? lo + PT : n;
  const u64 ll = m <= lo ? 0 : (m >= hi ? hi - lo : m - lo);  // words left of m
  const u64 tleft = k < kb ? tck : (k == kb ? tl : 0);          // true words left of m
  ml = ll - tleft;
  mr = tck - tleft;
}

__device__ __forceinline__ u64 block_sum_u64(u64 v, u64* s_red) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_down_sync(0xffffffffu, v, o);
  const u32 w = threadIdx.x >> 5, nw = blockDim.x >> 5;
  if ((threadIdx.x & 31) == 0) s_red[w] = v;
  __syncthreads();
  u64 t = 0;
  for (u32 i = 0; i < nw; ++i) t += s_red[i];
  __syncthreads();
  return t;
}

// inclusive block scan of two u64 values (Hillis-Steele over warps' totals)
__device__ __forceinline__ void block_scan2(u64& a, u64& b, u64* s_a, u64* s_b, u64& ta, u64& tb) {
  const u32 lane = threadIdx.x & 31, w = threadIdx.x >> 5, nw = blockDim.x >> 5;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const u64 xa = __shfl_up_sync(0xffffffffu, a, o), xb = __shfl_up_sync(0xffffffffu, b, o);
    if (lane >= (u32)o) { a += xa; b += xb; }
  }
  if (lane == 31) { s_a[w] = a; s_b[w] = b; }
  __syncthreads();
  u64 pa = 0, pb = 0;
  ta = 0;
  tb = 0;
  for (u32 i = 0; i < nw; ++i) {
    if (i < w) { pa += s_a[i]; pb += s_b[i]; }
    ta += s_a[i];
    tb += s_b[i];
  }
  a += pa;
  b += pb;
  __syncthreads();
}

__device__ __forceinline__ void group_range(u64 g, u64 ntiles, u64 G, u64& k0, u64& k1) {
  const u64 per = (ntiles + G - 1) / G;
  k0 = g * per < ntiles ? g * per : ntiles;
  k1 = k0 + per < ntiles ? k0 + per : ntiles;
}

__global__ void __launch_bounds__(PL_THREADS) part_gsum_kernel(const u32* __restrict__ tc, u64 ntiles,
                                                               u64* gsum) {
  __shared__ u64 s_red[PL_THREADS / 32];
  u64 k0, k1;
  group_range(blockIdx.x, ntiles, gridDim.x, k0, k1);
  u64 s = 0;
  for (u64 k = k0 + threadIdx.x; k < k1; k += PL_THREADS) s += __ldcg(tc + k);
  s = block_sum_u64(s, s_red);
  if (threadIdx.x == 0) gsum[blockIdx.x] = s;
}

template <int PC>
__global__ void __launch_bounds__(PL_THREADS) part_plan_kernel(const u64* __restrict__ a, u64 n,
                                                               DevPred p, const u32* __restrict__ tc,
                                                               u64 ntiles, u64 G, u64* gsum,
                                                               PartInfo* info, u64* m_dev) {
  // gsum[g] in: true words of group g; out: (misL base, misR base) in gsum[g], gsum[PL_GROUPS + g]
  __shared__ u64 s_a[PL_THREADS / 32], s_b[PL_THREADS / 32];
  __shared__ u32 s_tl;
  const u32 t = threadIdx.x;  // == group (groups >= G are empty)
  const u64 gs = t < G ? __ldcg(gsum + t) : 0ull;
  const u64 m = block_sum_u64(gs, s_a);
  const u64 kb = m / PT;
  if (t == 0) s_tl = 0;
  __syncthreads();
  if (kb < ntiles) {
    u32 c = 0;
    for (u64 i = kb * PT + t; i < m; i += PL_THREADS) c += (u32)pred_eval_t<PC>(p, a[i]);
    c = __reduce_add_sync(0xffffffffu, c);
    if ((t & 31) == 0 && c) atomicAdd(&s_tl, c);
  }
  __syncthreads();
  const u32 tl = s_tl;
  // misfit sums of group t: closed forms unless the group holds tile kb
  u64 k0 = ntiles, k1 = ntiles;
  if (t < G) group_range(t, ntiles, G, k0, k1);
  u64 ml = 0, mr = 0;
  const u64 w0 = k0 * PT < n ? k0 * PT : n, w1 = k1 * PT < n ? k1 * PT : n;
  if (k0 == k1) {
  } else if (k1 <= kb) {
    ml = (w1 - w0) - gs;
  } else if (k0 > kb) {
    mr = gs;
  } else {
    for (u64 k = k0; k < k1; ++k) {
      u64 a1, b1;
      tile_mis(k, n, m, kb, tl, __ldcg(tc + k), a1, b1);
      ml += a1;
      mr += b1;
    }
  }
  u64 il = ml, ir = mr, tot_l, tot_r;
  block_scan2(il, ir, s_a, s_b, tot_l, tot_r);
  if (t < G) {
    gsum[t] = il - ml;
    gsum[G + t] = ir - mr;
  }
  if (t == 0) {
    info->m = m;
    info->X = tot_l;  // == tot_r
    info->kb = kb;
    info->nleft = (m + PT - 1) / PT;
    info->tl = tl;
    *m_dev = m;
  }
}

__global__ void __launch_bounds__(PL_THREADS) part_base_kernel(const u32* __restrict__ tc, u64 n,
                                                               u64 ntiles, const u64* __restrict__ gsum,
                                                               const PartInfo* info, u64* baseL,
                                                               u64* baseR) {
  __shared__ u64 s_a[PL_THREADS / 32], s_b[PL_THREADS / 32];
  const u64 m = info->m, kb = info->kb;
  const u32 tl = (u32)info->tl;
  u64 k0, k1;
  group_range(blockIdx.x, ntiles, gridDim.x, k0, k1);
  u64 bl = gsum[blockIdx.x], br = gsum[gridDim.x + blockIdx.x];
  for (u64 c0 = k0; c0 < k1; c0 += PL_THREADS) {
    const u64 k = c0 + threadIdx.x;
    u64 ml = 0, mr = 0;
    if (k < k1) tile_mis(k, n, m, kb, tl, __ldcg(tc + k), ml, mr);
    u64 il = ml, ir = mr, tl_, tr_;
    block_scan2(il, ir, s_a, s_b, tl_, tr_);
    if (k < k1) {
      baseL[k] = bl + il - ml;
      baseR[k] = br + ir - mr;
    }
    bl += tl_;
    br += tr_;
  }
}

// ---------------------------------------------------------------- K3 bounds
// one warp per left tile k with misfits: position of right misfit rank baseL[k]
template <int PC>
__global__ void __launch_bounds__(256) part_bounds_kernel(const u64* __restrict__ a, u64 n, DevPred p,
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
    // right tile j: largest j in [kb, ntiles) with baseR[j] <= r, i.e. the
    // first j' in (kb, ntiles] with baseR[j'] > r, minus one; gallop from
    // the proportional estimate (misfits spread over the right tiles)
    u64 lo = kb + 1, hi = ntiles;
    {
      u64 g = kb + (u64)(((unsigned __int128)r * (ntiles - kb)) / X);
      g = g < lo ? lo : (g >= hi ? (hi > lo ? hi - 1 : lo) : g);
      u64 st = 4;
      if (lo < hi) {
        if (__ldcg(baseR + g) <= r) {
          lo = g + 1;
          for (; lo + st <= hi; st <<= 1) {
            if (__ldcg(baseR + lo + st - 1) <= r) lo += st;
            else { hi = lo + st - 1; break; }
          }
        } else {
          hi = g;
          for (; hi >= lo + st; st <<= 1) {
            if (!(__ldcg(baseR + hi - st) <= r)) hi -= st;
            else { lo = hi - st + 1; break; }
          }
        }
      }
      while (lo < hi) {
        const u64 mid = (lo + hi) >> 1;
        if (__ldcg(baseR + mid) <= r) lo = mid + 1;
        else hi = mid;
      }
    }
    const u64 j = lo - 1;
    u64 q = r - __ldcg(baseR + j);  // rank inside tile j
    const u64 s0 = j * PT > m ? j * PT : m, s1 = (j + 1) * PT < n ? (j + 1) * PT : n;
    u64 pos = ~0ull;
    // 8 consecutive words per lane, 256 per step
    for (u64 i0 = s0; i0 < s1; i0 += 256) {
      u32 bits = 0;
#pragma unroll
      for (int z = 0; z < 8; ++z) {
        const u64 i = i0 + (u64)lane * 8 + z;
        bits |= (u32)(i < s1 && pred_eval_t<PC>(p, i < s1 ? a[i] : 0ull)) << z;
      }
      const u32 c = __popc(bits);
      u32 x = c;  // inclusive warp prefix
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const u32 y = __shfl_up_sync(0xffffffffu, x, o);
        if (lane >= (u32)o) x += y;
      }
      const u32 tot = __shfl_sync(0xffffffffu, x, 31);
      if (q < tot) {
        // the lane whose inclusive prefix first exceeds q holds it
        const unsigned hit = __ballot_sync(0xffffffffu, x > q);
        const u32 L = (u32)(__ffs(hit) - 1);
        if (lane == L) {
          u32 b = bits;
          for (u32 z = 0, need = (u32)q - (x - c); z < need; ++z) b &= b - 1;
          pos = i0 + (u64)lane * 8 + (u64)(__ffs(b) - 1);
        }
        pos = __shfl_sync(0xffffffffu, pos, L);
        break;
      }
      q -= tot;
    }
    if (lane == 0) startR[k] = pos;
  }
}

// ---------------------------------------------------------------- K4 swap
struct PartSmem {
  u64 lval[PT];
  u64 rval[PT];
  u32 rpos[PT];  // offset from startR[k]
  unsigned short lpos[PT];
  u32 cnt_l;
  u32 warp[PT_THREADS / 32];
};

template <int PC>
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
    // left misfits: false words of [kT, min((k+1)T, m)) (pairing order is free)
    if (tid == 0) S.cnt_l = 0;
    __syncthreads();
    const u64 lo = k * PT, hi = lo + PT < m ? lo + PT : m;
    u64 lv[PT_PER];
#pragma unroll
    for (int q = 0; q < PT_PER; ++q) {
      const u64 i = lo + tid + (u64)q * PT_THREADS;
      lv[q] = i < hi ? a[i] : 0ull;
    }
#pragma unroll
    for (int q = 0; q < PT_PER; ++q) {
      const u64 i = lo + tid + (u64)q * PT_THREADS;
      if (i < hi && !pred_eval_t<PC>(p, lv[q])) {
        const u32 s = atomicAdd(&S.cnt_l, 1u);
        S.lval[s] = lv[q];
        S.lpos[s] = (unsigned short)(i - lo);
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
      }
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        f[q] = i0 + (u64)tid * 4 + q < n && pred_eval_t<PC>(p, v[q]);
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
#pragma unroll
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

// ---------------------------------------------------------------- leaf sort
// quicksort leaves (strong.quicksort_strong's base case a[lo:hi].sort(),
// strong.py:453-454): one CTA per segment of <= 2^20 words.  Bitonic sort
// in its all-ascending "flip" form: every compare-exchange puts the max at
// the higher index, so the virtual +inf padding above the segment's length
// never moves and partners past the end are simply skipped.  Stages whose
// pairs lie inside an aligned 8192-word chunk run in shared memory (one
// chunk at a time); the wider flip / half-cleaner stages of segments longer
// than one chunk run on global memory (L2-resident: the CTA owns the
// segment, __syncthreads orders the passes).
static constexpr u32 SEG_CHUNK = 8192;
static constexpr u32 SEG_MAX = 1u << 20;
static constexpr u64 SEG_MAX_GRID = 1ull << 28;

__device__ __forceinline__ void cas_smem(u64* ss, u32 l, u32 r) {
  const u64 x = ss[l], y = ss[r];
  if (x > y) {
    ss[l] = y;
    ss[r] = x;
  }
}

// stages [k0 .. C] of the flip network on one chunk in shared memory
// (k0 = 2: full local sort; k0 > C: only the half-cleaners below C)
__device__ void seg_chunk_pass(u64* base, u32 c0, u32 L, u32 C, u32 k_lo, u32 k_hi, u64* ss) {
  const u32 tid = threadIdx.x;
  for (u32 i = tid; i < C; i += 1024) ss[i] = c0 + i < L ? base[c0 + i] : ~0ull;
  __syncthreads();
  for (u32 k = k_lo; k <= k_hi; k <<= 1) {
    const u32 half = k >> 1;
    for (u32 i = tid; i < C / 2; i += 1024) {
      const u32 pos = i & (half - 1), blk = (i - pos) << 1;
      cas_smem(ss, blk + pos, blk + k - 1 - pos);
    }
    __syncthreads();
    for (u32 j = k >> 2; j > 0; j >>= 1) {
      for (u32 i = tid; i < C / 2; i += 1024) {
        const u32 l = 2 * i - (i & (j - 1));
        cas_smem(ss, l, l + j);
      }
      __syncthreads();
    }
  }
  if (k_lo > k_hi) {  // half-cleaners j = C/2 .. 1 only
    for (u32 j = C >> 1; j > 0; j >>= 1) {
      for (u32 i = tid; i < C / 2; i += 1024) {
        const u32 l = 2 * i - (i & (j - 1));
        cas_smem(ss, l, l + j);
      }
      __syncthreads();
    }
  }
  for (u32 i = tid; c0 + i < L && i < C; i += 1024) base[c0 + i] = ss[i];
  __syncthreads();
}

__device__ __forceinline__ void cas_glob(u64* base, u32 l, u32 r, u32 L) {
  if (r < L) {
    const u64 x = base[l], y = base[r];
    if (x > y) {
      base[l] = y;
      base[r] = x;
    }
  }
}

__global__ void __launch_bounds__(1024) segsort_kernel(u64* a, const u64* __restrict__ seg_lo,
                                                       const u32* __restrict__ seg_len, u64 nseg) {
  extern __shared__ __align__(16) u64 ss[];
  const u32 tid = threadIdx.x;
  for (u64 g = blockIdx.x; g < nseg; g += gridDim.x) {
    const u32 L = seg_len[g];
    if (L < 2) continue;
    u64* base = a + seg_lo[g];
    u32 P = 2;
    while (P < L) P <<= 1;
    const u32 C = P < SEG_CHUNK ? P : SEG_CHUNK;
    for (u32 c0 = 0; c0 < L; c0 += C) seg_chunk_pass(base, c0, L, C, 2, C, ss);
    for (u32 k = 2 * C; k <= P; k <<= 1) {
      const u32 half = k >> 1;
      for (u32 i = tid; i < P / 2; i += 1024) {
        const u32 pos = i & (half - 1), blk = (i - pos) << 1;
        cas_glob(base, blk + pos, blk + k - 1 - pos, L);
      }
      __syncthreads();
      for (u32 j = k >> 2; j >= C; j >>= 1) {
        for (u32 i = tid; i < P / 2; i += 1024) {
          const u32 l = 2 * i - (i & (j - 1));
          cas_glob(base, l, l + j, L);
        }
        __syncthreads();
      }
      for (u32 c0 = 0; c0 < L; c0 += C) seg_chunk_pass(base, c0, L, C, 2 * C, C, ss);
    }
  }
}

// The same network spread over the grid (for leaves longer than one chunk):
// blockIdx.x = segment, blockIdx.y = chunk / pair range inside it.  One
// launch sorts every chunk of every segment locally, then each wider stage
// k is one launch for the flip stage, one per half-cleaner distance >= one
// chunk, and one for the chunk-local cleaners -- every SM busy whatever the
// number of segments.
__device__ __forceinline__ u32 seg_pow2(u32 L) {
  u32 P = 2;
  while (P < L) P <<= 1;
  return P;
}

__global__ void __launch_bounds__(1024) segsort_local_kernel(u64* a, const u64* __restrict__ seg_lo,
                                                             const u32* __restrict__ seg_len, u32 k) {
  extern __shared__ __align__(16) u64 ss[];
  const u32 L = seg_len[blockIdx.x];
  if (L < 2) return;
  const u32 P = seg_pow2(L);
  const u32 C = P < SEG_CHUNK ? P : SEG_CHUNK;
  const u32 c0 = blockIdx.y * C;
  if (c0 >= L) return;
  if (k == 0) {
    seg_chunk_pass(a + seg_lo[blockIdx.x], c0, L, C, 2, C, ss);
  } else if (k <= P) {
    seg_chunk_pass(a + seg_lo[blockIdx.x], c0, L, C, 2 * C, C, ss);
  }
}

__global__ void __launch_bounds__(1024) segsort_global_kernel(u64* a, const u64* __restrict__ seg_lo,
                                                              const u32* __restrict__ seg_len, u32 k,
                                                              u32 j) {
  const u32 L = seg_len[blockIdx.x];
  if (L < 2) return;
  const u32 P = seg_pow2(L);
  if (k > P) return;
  const u32 i0 = blockIdx.y * (SEG_CHUNK / 2);
  if (i0 >= P / 2) return;
  u64* base = a + seg_lo[blockIdx.x];
  const u32 half = k >> 1;
  for (u32 i = i0 + threadIdx.x; i < i0 + SEG_CHUNK / 2; i += 1024) {
    if (j == 0) {
      const u32 pos = i & (half - 1), blk = (i - pos) << 1;
      cas_glob(base, blk + pos, blk + k - 1 - pos, L);
    } else {
      const u32 l = 2 * i - (i & (j - 1));
      cas_glob(base, l, l + j, L);
    }
  }
}

int sort_segments_grid_device(u64* a, const u64* seg_lo, const u32* seg_len, u64 nseg,
                              u64 max_len, cudaStream_t st) {
  if (nseg == 0) return PIP_OK;
  if (!a || !seg_lo || !seg_len || max_len > SEG_MAX_GRID || nseg > 0x7fffffffull)
    return PIP_ERR_INVALID_ARG;
  u32 Pmax = 2;
  while (Pmax < max_len) Pmax <<= 1;
  const size_t smem = SEG_CHUNK * 8;
  PIP_CUDA(cudaFuncSetAttribute(segsort_local_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                (int)smem));
  const u32 C = Pmax < SEG_CHUNK ? Pmax : SEG_CHUNK;
  const dim3 grid((unsigned)nseg, Pmax / C);
  segsort_local_kernel<<<grid, 1024, smem, st>>>(a, seg_lo, seg_len, 0);
  PIP_CHECK_LAUNCH();
  for (u32 k = 2 * SEG_CHUNK; k <= Pmax; k <<= 1) {
    segsort_global_kernel<<<grid, 1024, 0, st>>>(a, seg_lo, seg_len, k, 0);
    PIP_CHECK_LAUNCH();
    for (u32 j = k >> 2; j >= SEG_CHUNK; j >>= 1) {
      segsort_global_kernel<<<grid, 1024, 0, st>>>(a, seg_lo, seg_len, k, j);
      PIP_CHECK_LAUNCH();
    }
    segsort_local_kernel<<<grid, 1024, smem, st>>>(a, seg_lo, seg_len, k);
    PIP_CHECK_LAUNCH();
  }
  return PIP_OK;
}

int sort_segments_device(u64* a, const u64* seg_lo, const u32* seg_len, u64 nseg, cudaStream_t st) {
  if (nseg == 0) return PIP_OK;
  if (!a || !seg_lo || !seg_len) return PIP_ERR_INVALID_ARG;
  const size_t smem = SEG_CHUNK * 8;
  PIP_CUDA(cudaFuncSetAttribute(segsort_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  const int sms = num_sms(current_device());
  const u64 g = nseg < (u64)sms * 3 ? nseg : (u64)sms * 3;
  segsort_kernel<<<(unsigned)g, 1024, smem, st>>>(a, seg_lo, seg_len, nseg);
  PIP_CHECK_LAUNCH();
  return PIP_OK;
}

// ---------------------------------------------------------------- host
// groups of tiles for the plan: one per 64 tiles, at most PL_GROUPS
static u64 part_groups(u64 ntiles) {
  const u64 g = (ntiles + 63) / 64;
  return g < 1 ? 1 : (g > (u64)PL_GROUPS ? (u64)PL_GROUPS : g);
}

struct PartLayout {
  size_t tc, baseL, baseR, startR, info, gsum, total;
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
  L.gsum = take(2 * part_groups(ntiles) * 8);
  L.total = off;
  return L;
}

size_t partition_workspace_bytes(u64 n) { return n ? part_layout(n).total : 0; }

template <int PC>
static int part_launch(u64* a, u64 n, const DevPred& p, u64* m_dev, u32* tc, u64* baseL, u64* baseR,
                       u64* startR, PartInfo* info, u64 ntiles, u64* gsum, cudaStream_t st) {
  const int sms = num_sms(current_device());
  const u64 g1 = ntiles < (u64)sms * 8 ? ntiles : (u64)sms * 8;
  part_count_kernel<PC><<<(unsigned)g1, PT_THREADS, 0, st>>>(a, n, p, tc, ntiles);
  PIP_CHECK_LAUNCH();
  const u64 G = part_groups(ntiles);
  part_gsum_kernel<<<(unsigned)G, PL_THREADS, 0, st>>>(tc, ntiles, gsum);
  PIP_CHECK_LAUNCH();
  part_plan_kernel<PC><<<1, PL_THREADS, 0, st>>>(a, n, p, tc, ntiles, G, gsum, info, m_dev);
  PIP_CHECK_LAUNCH();
  part_base_kernel<<<(unsigned)G, PL_THREADS, 0, st>>>(tc, n, ntiles, gsum, info, baseL, baseR);
  PIP_CHECK_LAUNCH();
  const u64 g3 = (ntiles + 7) / 8 < (u64)sms * 8 ? (ntiles + 7) / 8 : (u64)sms * 8;
  part_bounds_kernel<PC><<<(unsigned)g3, 256, 0, st>>>(a, n, p, baseL, baseR, ntiles, info, startR);
  PIP_CHECK_LAUNCH();
  const size_t smem = sizeof(PartSmem);
  PIP_CUDA(cudaFuncSetAttribute(part_swap_kernel<PC>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                (int)smem));
  const u64 g4 = ntiles < (u64)sms * 4 ? ntiles : (u64)sms * 4;
  part_swap_kernel<PC><<<(unsigned)g4, PT_THREADS, smem, st>>>(a, n, p, baseL, ntiles, info, startR);
  PIP_CHECK_LAUNCH();
  return PIP_OK;
}

int partition_device(u64* a, u64 n, const pip_pred* pred, u64* m_dev, void* ws, size_t ws_bytes,
                     cudaStream_t st) {
  if (!pred || !m_dev || pred->kind > PIP_PRED_EQ) return PIP_ERR_INVALID_ARG;
  if (pred->kind == PIP_PRED_MOD_EQ && pred->a == 0) return PIP_ERR_INVALID_ARG;
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
  u64* gsum = (u64*)(w + L.gsum);
  const u64 ntiles = (n + PT - 1) / PT;
  const DevPred p = make_dev_pred(*pred);
  switch (part_pred_class(p)) {
    case PC_MASK: return part_launch<PC_MASK>(a, n, p, m_dev, tc, baseL, baseR, startR, info, ntiles, gsum, st);
    case PC_MOD: return part_launch<PC_MOD>(a, n, p, m_dev, tc, baseL, baseR, startR, info, ntiles, gsum, st);
    case PC_MODODD: return part_launch<PC_MODODD>(a, n, p, m_dev, tc, baseL, baseR, startR, info, ntiles, gsum, st);
    case PC_MODODD0: return part_launch<PC_MODODD0>(a, n, p, m_dev, tc, baseL, baseR, startR, info, ntiles, gsum, st);
    default: return part_launch<PC_GEN>(a, n, p, m_dev, tc, baseL, baseR, startR, info, ntiles, gsum, st);
  }
}

}  // namespace pip
