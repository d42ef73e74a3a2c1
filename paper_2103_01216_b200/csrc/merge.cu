// In-place merge of two sorted runs (strong.merge_strong,
// relaxed.merge_relaxed).
//
// Reference: pkg/src/pipal/strong.py:462-522 (co-rank by dual binary search
// `_split_point` :474-488, rotate the middle by triple reversal, recurse:
// O(n log n) moves) and pkg/src/pipal/relaxed.py:377-612 (k = b(n) chunks:
// descriptor sort of chunks by their last element :509-527, whole-chunk
// cycle permutation through a k-word buffer :531-546, three-chunk streaming
// merge :413-506, tails parked and merged back :566-612).
//
// B200 design — two streaming passes over HBM, both fully parallel:
//   P0  (descriptors, O(n/C) work) chunks of C = 8192 words; A' = the A
//       words after its head A[0:hA) (hA = |A| mod C), B' = the B words
//       before its tail (hB = |B| mod C), so A' and B' are whole chunks of
//       one contiguous slot region [hA, n - hB); the head and the tail stay
//       where they are.  Every chunk gets its destination slot in the order
//       of chunk LAST elements (the reference's descriptor sort, ties A
//       before B), and the merge-path co-ranks of every output block
//       [mC, (m+1)C) over the original runs A, B are computed BEFORE
//       anything moves.
//   P1  (chunk permutation, ~16 B/word) the slot permutation is applied in
//       place by walking its cycles backwards from "cut" slots whose chunks
//       were first saved to a cut buffer (cuts every D slots — D set by the
//       workspace budget); every walk is independent, so all CTAs walk in
//       parallel; cycles that contain no cut (rare) are found by pointer
//       jumping (min-label) and rotated by one CTA each through shared
//       memory.
//   P2  (block merge, ~16 B/word) after the permutation a chunk in slot q
//       only holds words of output rank < (q+2)C + hA + hB (chunks sorted by
//       last element), so output block m can be written as soon as every
//       block <= m + L (L = 1 + ceil((hA+hB)/C)) has loaded its inputs.
//       (Block m's region overlaps slots <= m; a word of the chunk in slot q
//       has fewer than qC + C + C + hA + hB words before it in the merged
//       order — the q chunks of smaller-or-equal last, its own chunk, one
//       partial chunk of the other run, head and tail — so it belongs to a
//       block <= q + 1 + ceil((hA+hB)/C).)
//       Blocks are assigned round-robin to persistent CTAs, loaded (<= 6
//       contiguous pieces) into shared memory, merged by merge path and
//       written back under that dataflow rule — no grid barrier per block.
//       Block 0 (the only writer of the in-place head) is kept in shared
//       memory and written after a final barrier; the blocks over the tail
//       are the last ones and wait for every load anyway.
// Output equals np.sort(a) (values are plain words, so the tie order is
// invisible; it is fixed here as A before B for the co-ranks).
#include <cstdio>
#include <cstdlib>
#include "sync.cuh"

namespace pip {

static constexpr int MG_THREADS = 512;
static constexpr int MG_CTAS_PER_SM = 1;
static constexpr u32 MG_LOGC = 13;
static constexpr u64 MG_C = 1ull << MG_LOGC;  // words per chunk / output block
static constexpr int MG_PER_THREAD = (int)(MG_C / MG_THREADS);
// shared-memory padding: merge-path readers sit ~8 words apart and writers
// exactly 16 words apart, which on 8-byte words means 16- and 32-way bank
// conflicts; one pad word per 8 (inputs) / per 16 (outputs) spreads them
__device__ __forceinline__ u32 SI(u32 l) { return l + (l >> 3); }
__device__ __forceinline__ u32 SO(u32 r) { return r + (r >> 4); }
static constexpr u32 MG_IN_WORDS = (u32)(MG_C + MG_C / 8);
static constexpr u32 MG_OUT_WORDS = (u32)(MG_C + MG_C / 16);
static constexpr u32 MG_STAGE_WORDS = (u32)(MG_C + 16);  // bulk-copy staging (+2 junk words x 6 segments)
static constexpr size_t MG_SMEM = (size_t)(2 * MG_STAGE_WORDS + MG_C) * 8;

struct MergeGlobal {
  GridSync sync;
  u32 walk_next;  // dynamic walk assignment
  u32 uncut;      // #slots on cut-free cycles
  u64 t[8];       // %globaltimer at phase boundaries (CTA 0)
  u64 sec[6];     // PIP_MERGE_DBG bit2: CTA 0 cycles in stage|load-issue|merge|wait|store|other
};

struct MergeArgs {
  u32 dbg;  // profiling knobs (PIP_MERGE_DBG): bit0 skip the dataflow wait, bit1 copy instead of merge
  u64* a;
  u64 n, na, nb;
  u64 hA, hB, KA, KB, K, NB, D, ncuts, L;
  u64* cut;       // [ncuts * C] saved chunks of the cut slots
  u32* dest;      // [K] destination slot of the chunk in slot s
  u32* inv;       // [K] slot whose chunk moves into slot s
  u32* lab[2];    // [K] pointer-jumping labels   (only if uncut cycles)
  u32* jmp[2];    // [K] pointer-jumping jumps
  unsigned char* visited;  // [K]
  u64* cr;        // [NB + 1] A co-rank of every output block boundary
  ulonglong4* plan;  // [NB] {i0, i1, dest slots of the <= 2 A' and <= 2 B' chunks}
  u32* status;    // [G] per CTA: (last block loaded) + 1
  MergeGlobal* g;
};

__device__ __forceinline__ void mpart(u64 total, u32 G, u32 b, u64& s, u64& e) {
  s = total * b / G;
  e = total * (b + 1) / G;
}

// physical word of A[x] / B[y] once the chunks sit in their destination
// slots (the head A[0:hA) and the tail B[nb-hB:nb) never move)
__device__ __forceinline__ u64 phys_a(const MergeArgs& M, u64 x) {
  if (x < M.hA) return x;
  const u64 xp = x - M.hA;
  return M.hA + ((u64)__ldcg(M.dest + (xp >> MG_LOGC)) << MG_LOGC) + (xp & (MG_C - 1));
}
__device__ __forceinline__ u64 phys_b(const MergeArgs& M, u64 y) {
  if (y >= M.nb - M.hB) return M.na + y;
  return M.hA + ((u64)__ldcg(M.dest + M.KA + (y >> MG_LOGC)) << MG_LOGC) + (y & (MG_C - 1));
}

// merge path over the original runs A = a[0:na), B = a[na:n) (A first on ties)
__device__ __forceinline__ u64 corank2_global(const MergeArgs& M, u64 q) {
  const u64* A = M.a;
  const u64* B = M.a + M.na;
  u64 lo = q > M.nb ? q - M.nb : 0, hi = q < M.na ? q : M.na;
  while (lo < hi) {
    const u64 mid = (lo + hi) >> 1;
    if (__ldcg(A + mid) <= __ldcg(B + (q - mid - 1))) lo = mid + 1;
    else hi = mid;
  }
  return lo;
}

// merge path over the padded input buffer: A = logical [0, na), B = [na, na + nb)
__device__ __forceinline__ u32 corank2_smem(const u64* s, u32 na, u32 nb, u32 q) {
  u32 lo = q > nb ? q - nb : 0, hi = q < na ? q : na;
  while (lo < hi) {
    const u32 mid = (lo + hi) >> 1;
    if (s[SI(mid)] <= s[SI(na + q - mid - 1)]) lo = mid + 1; else hi = mid;
  }
  return lo;
}

// merge A and B of the padded input `s` into the padded output `out`;
// MG_PER_THREAD outputs per thread from its merge-path co-rank; one shared
// load per output (the consumed side's next key), no data-dependent branches
__device__ __forceinline__ void block_merge(const u64* s, u32 na, u32 nb, u64* out) {
  const u32 total = na + nb;
  const u32 r0 = threadIdx.x * MG_PER_THREAD;
  if (r0 >= total) return;
  u32 i = corank2_smem(s, na, nb, r0);
  u32 j = r0 - i;
  u64 ka = i < na ? s[SI(i)] : ~0ull;
  u64 kb = j < nb ? s[SI(na + j)] : ~0ull;
  const u32 r1 = r0 + MG_PER_THREAD < total ? r0 + MG_PER_THREAD : total;
#pragma unroll 4
  for (u32 r = r0; r < r1; ++r) {
    const bool pa = (j >= nb) || (i < na && ka <= kb);  // ties from A
    out[SO(r)] = pa ? ka : kb;
    const u32 ni = i + (pa ? 1u : 0u), nj = j + (pa ? 0u : 1u);
    const bool more = pa ? (ni < na) : (nj < nb);
    const u64 nk = more ? s[SI(pa ? ni : na + nj)] : ~0ull;
    ka = pa ? nk : ka;
    kb = pa ? kb : nk;
    i = ni;
    j = nj;
  }
}

__device__ __forceinline__ bool is_cut(const MergeArgs& M, u64 s) {
  return M.ncuts && (s % M.D) == 0 && __ldcg(M.inv + s) != (u32)s;
}

// copy one chunk, whole CTA (8-byte accesses: slots start at hA, which need
// not be 16-byte aligned); every thread reads before anyone writes
__device__ __forceinline__ void move_chunk(u64* dst, const u64* src) {
  const u32 tid = threadIdx.x;
  u64 v[MG_PER_THREAD];
#pragma unroll
  for (int k = 0; k < MG_PER_THREAD; ++k) v[k] = __ldcg(src + tid + k * MG_THREADS);
  __syncthreads();
#pragma unroll
  for (int k = 0; k < MG_PER_THREAD; ++k) dst[tid + k * MG_THREADS] = v[k];
}

__device__ __forceinline__ u64* slot_ptr(const MergeArgs& M, u64 s) {
  return M.a + M.hA + (s << MG_LOGC);
}

__global__ void __launch_bounds__(MG_THREADS, MG_CTAS_PER_SM) merge_kernel(MergeArgs M) {
  extern __shared__ __align__(16) u64 smem[];
  u64* s_out = smem;  // P1b: one chunk in transit
  __shared__ u64 s_misc[2];
  __shared__ int s_flag;
  const u32 b = blockIdx.x, G = gridDim.x, tid = threadIdx.x;
  MergeGlobal* g = M.g;
  u32 gen = 0;
  u64* a = M.a;
  const bool tm = b == 0 && tid == 0;
  if (tm) g->t[0] = globaltimer_ns();

  // ---------------- P0: slot destinations (sort by chunk last) + co-ranks
  {
    u64 s, e;
    mpart(M.K, G, b, s, e);
    for (u64 x = s + tid; x < e; x += MG_THREADS) {
      u64 d;
      if (x < M.KA) {
        const u64 last = __ldcg(a + M.hA + ((x + 1) << MG_LOGC) - 1);
        u64 lo = 0, hi = M.KB;  // #B' chunks with last < this last
        while (lo < hi) {
          const u64 mid = (lo + hi) >> 1;
          if (__ldcg(a + M.na + ((mid + 1) << MG_LOGC) - 1) < last) lo = mid + 1; else hi = mid;
        }
        d = x + lo;
      } else {
        const u64 y = x - M.KA;
        const u64 last = __ldcg(a + M.na + ((y + 1) << MG_LOGC) - 1);
        u64 lo = 0, hi = M.KA;  // #A' chunks with last <= this last
        while (lo < hi) {
          const u64 mid = (lo + hi) >> 1;
          if (__ldcg(a + M.hA + ((mid + 1) << MG_LOGC) - 1) <= last) lo = mid + 1; else hi = mid;
        }
        d = y + lo;
      }
      M.dest[x] = (u32)d;
      M.inv[d] = (u32)x;
      M.visited[x] = 0;
    }
    mpart(M.NB + 1, G, b, s, e);
    for (u64 m = s + tid; m < e; m += MG_THREADS) {
      const u64 p = m * MG_C < M.n ? m * MG_C : M.n;
      M.cr[m] = corank2_global(M, p);
    }
  }
  if (!grid_barrier(&g->sync, gen)) return;
  if (tm) g->t[1] = globaltimer_ns();

  // ---------------- P0b: per-block load plans; save the chunks of the cut slots
  {
    u64 s, e;
    mpart(M.NB, G, b, s, e);
    const u64 lb = M.nb - M.hB;
    for (u64 m = s + tid; m < e; m += MG_THREADS) {
      const u64 p0 = m * MG_C, p1 = (m + 1) * MG_C < M.n ? (m + 1) * MG_C : M.n;
      const u64 i0 = __ldcg(M.cr + m), i1 = __ldcg(M.cr + m + 1);
      const u64 j0 = p0 - i0, j1 = p1 - i1;
      u32 da0 = 0, da1 = 0, db0 = 0, db1 = 0;
      const u64 xs = i0 > M.hA ? i0 : M.hA;
      if (xs < i1) {
        da0 = __ldcg(M.dest + ((xs - M.hA) >> MG_LOGC));
        da1 = __ldcg(M.dest + ((i1 - 1 - M.hA) >> MG_LOGC));
      }
      const u64 ye = j1 < lb ? j1 : lb;
      if (j0 < ye) {
        db0 = __ldcg(M.dest + M.KA + (j0 >> MG_LOGC));
        db1 = __ldcg(M.dest + M.KA + ((ye - 1) >> MG_LOGC));
      }
      M.plan[m] = make_ulonglong4(i0, i1, ((u64)da1 << 32) | da0, ((u64)db1 << 32) | db0);
    }
  }
  for (u64 c = b; c < M.ncuts; c += G) {
    const u64 slot = c * M.D;
    if (__ldcg(M.inv + slot) != (u32)slot) move_chunk(M.cut + c * MG_C, slot_ptr(M, slot));
    __syncthreads();
  }
  if (!grid_barrier(&g->sync, gen)) return;
  if (tm) g->t[2] = globaltimer_ns();

  // ---------------- P1: chunk permutation: walk each cycle backwards from a cut
  for (;;) {
    if (tid == 0) s_misc[0] = atomicAdd(&g->walk_next, 1u);
    __syncthreads();
    const u64 c = s_misc[0];
    __syncthreads();
    if (c >= M.ncuts) break;
    const u64 p0 = c * M.D;
    if (__ldcg(M.inv + p0) == (u32)p0) continue;
    u64 sdst = p0;
    for (u64 steps = 0; steps <= M.K; ++steps) {
      const u64 src = __ldcg(M.inv + sdst);
      const bool last = is_cut(M, src);
      move_chunk(slot_ptr(M, sdst), last ? M.cut + (src / M.D) * MG_C : slot_ptr(M, src));
      if (tid == 0) M.visited[sdst] = 1;
      if (last) break;
      sdst = src;
    }
    __syncthreads();
  }
  if (!grid_barrier(&g->sync, gen)) return;
  if (tm) g->t[3] = globaltimer_ns();

  // ---------------- P1b: cycles without a cut (rare; all of them if no cut buffer)
  {
    u64 s, e;
    mpart(M.K, G, b, s, e);
    u32 cnt = 0;
    for (u64 x = s + tid; x < e; x += MG_THREADS)
      cnt += !__ldcg(M.visited + x) && __ldcg(M.inv + x) != (u32)x;
    cnt = __reduce_add_sync(0xffffffffu, cnt);
    if ((tid & 31) == 0 && cnt) atomicAdd(&g->uncut, cnt);
  }
  if (!grid_barrier(&g->sync, gen)) return;
  if (ld_relaxed_u32(&g->uncut)) {
    u64 s, e;
    mpart(M.K, G, b, s, e);
    for (u64 x = s + tid; x < e; x += MG_THREADS) {
      M.lab[0][x] = (u32)x;
      M.jmp[0][x] = __ldcg(M.inv + x);
    }
    if (!grid_barrier(&g->sync, gen)) return;
    // min-label by pointer jumping: after r rounds lab = min over 2^r steps
    u32 cur = 0;
    for (u64 span = 1; span < M.K; span <<= 1) {
      for (u64 x = s + tid; x < e; x += MG_THREADS) {
        const u32 j = __ldcg(M.jmp[cur] + x);
        const u32 l1 = __ldcg(M.lab[cur] + x), l2 = __ldcg(M.lab[cur] + j);
        M.lab[cur ^ 1][x] = l1 < l2 ? l1 : l2;
        M.jmp[cur ^ 1][x] = __ldcg(M.jmp[cur] + j);
      }
      cur ^= 1;
      if (!grid_barrier(&g->sync, gen)) return;
    }
    // each leader (cycle minimum) rotates its cycle through shared memory
    for (u64 x0 = b; x0 < M.K; x0 += G) {
      const bool lead = !__ldcg(M.visited + x0) && __ldcg(M.inv + x0) != (u32)x0 &&
                        __ldcg(M.lab[cur] + x0) == (u32)x0;
      if (!lead) continue;
      for (u32 k = tid; k < MG_C; k += MG_THREADS) s_out[k] = __ldcg(slot_ptr(M, x0) + k);
      __syncthreads();
      u64 sdst = x0;
      for (u64 steps = 0; steps <= M.K; ++steps) {
        const u64 src = __ldcg(M.inv + sdst);
        if (src == x0) {
          for (u32 k = tid; k < MG_C; k += MG_THREADS) slot_ptr(M, sdst)[k] = s_out[k];
          break;
        }
        move_chunk(slot_ptr(M, sdst), slot_ptr(M, src));
        sdst = src;
      }
      __syncthreads();
    }
    if (!grid_barrier(&g->sync, gen)) return;
  }

  if (tm) g->t[4] = globaltimer_ns();
  // ---------------- P2: block merge under the dataflow rule
  // Warp-specialized: warp 0 is the control warp, warps 1..15 merge.
  //   load   (control) the <= 6 contiguous input segments of a block (A head
  //          in place, <= 2 permuted A' chunks, <= 2 permuted B' chunks, B
  //          tail in place), one bulk copy each into one of two staging
  //          buffers, widened to 16-byte alignment (<= 2 junk words per
  //          segment); "loaded" is published as soon as the bytes land;
  //   merge  (merge warps) straight from staging through the segment map,
  //          a merge-path range of 17-18 consecutive outputs per thread into
  //          registers (ranges start at t*8192/480, not a multiple of 16
  //          words, so a warp's shared accesses spread over the banks even
  //          for perfectly interleaved runs); the staging buffer is handed
  //          back at once, the registers go to the output buffer as soon as
  //          the previous block's store has read it;
  //   store  (control) one bulk copy of the output buffer to a[mC, (m+1)C)
  //          once every block <= m + L has loaded (the dataflow rule).
  // The dataflow wait of block m overlaps the merge of block m + G.
  constexpr u32 NMW = MG_THREADS - 32;  // merge threads
  constexpr int MO = (int)((MG_C + NMW - 1) / NMW) + 1;  // outputs per thread, at most
  static_assert((2 * MG_STAGE_WORDS + MG_C) * 8 <= MG_SMEM, "two staging buffers + output");
  u64* s_obuf = smem + 2 * MG_STAGE_WORDS;
  __shared__ __align__(8) u64 s_full[2], s_sfree[2], s_ofull, s_ofree;
  __shared__ u32 s_seg[2][2 + 2 * 6];  // per buffer: na, nb | lo[6] | staging index[6]
  // CTA 0 keeps block 0's output (it overwrites the in-place head, which any
  // block may still read) in s_obuf to the end; its later blocks are written
  // back into their own staging buffer and stored from there
  const bool keep0 = M.hA > 0 && b == 0;
  const u64 nblk = b < M.NB ? (M.NB - 1 - b) / G + 1 : 0;  // blocks of this CTA
  auto in_place = [&](u64 j) { return keep0 && j > 0; };
  auto wait_or_abort = [&](u64* bar, u32 ph) -> bool {
    u32 n = 0;
    while (!mbar_try(bar, ph))
      if ((++n & 255) == 0 && ld_relaxed_u32(&g->sync.abort)) return false;
    return true;
  };
  if (tid == 0) {
    for (int q = 0; q < 2; ++q) {
      mbar_init(&s_full[q], 1);
      mbar_init(&s_sfree[q], 1);
    }
    mbar_init(&s_ofull, 1);
    mbar_init(&s_ofree, 1);
    mbar_fence_init();
  }
  __syncthreads();

  const bool prof = (M.dbg & 4) && b == 0 && (tid == 0 || tid == 32);
  u64 cyc[6] = {0, 0, 0, 0, 0, 0};
  u64 c0 = clock64();
  auto mark = [&](int q) {
    if (prof) {
      const u64 c1 = clock64();
      cyc[q] += c1 - c0;
      c0 = c1;
    }
  };

  if (tid < 32) {
    // ================================================= control warp
    const u32 lane = tid;
    ulonglong2 rec_a = make_ulonglong2(0, 0), rec_b = make_ulonglong2(0, 0);
    auto fetch_plan = [&](u64 m) {
      if (m < M.NB) {
        rec_a = __ldcg(reinterpret_cast<const ulonglong2*>(M.plan + m));
        rec_b = __ldcg(reinterpret_cast<const ulonglong2*>(M.plan + m) + 1);
      }
    };
    // lane k computes segment k: 0 A head, 1-2 A' pieces, 3-4 B' pieces, 5 B tail
    auto issue_load = [&](u64 m, int sb) {
      u64* stage = smem + sb * MG_STAGE_WORDS;
      const u64 p0 = m * MG_C, p1 = (m + 1) * MG_C < M.n ? (m + 1) * MG_C : M.n;
      const u64 i0 = rec_a.x, i1 = rec_a.y;
      const u32 da0 = (u32)rec_b.x, da1 = (u32)(rec_b.x >> 32);
      const u32 db0 = (u32)rec_b.y, db1 = (u32)(rec_b.y >> 32);
      fetch_plan(m + G);
      const u64 j0 = p0 - i0, j1 = p1 - i1;
      u64 ph = 0, len = 0;
      if (lane == 0) {  // A head [i0, min(i1, hA))
        const u64 xh = i1 < M.hA ? i1 : M.hA;
        if (i0 < xh) { ph = i0; len = xh - i0; }
      } else if (lane == 1 || lane == 2) {  // A' pieces
        const u64 xs = i0 > M.hA ? i0 : M.hA;
        if (xs < i1) {
          const u64 ce = M.hA + (((xs - M.hA) >> MG_LOGC) + 1) * MG_C;  // end of first chunk
          const u64 s0 = lane == 1 ? xs : ce, e0 = lane == 1 ? (ce < i1 ? ce : i1) : i1;
          if (s0 < e0) {
            ph = M.hA + ((u64)(lane == 1 ? da0 : da1) << MG_LOGC) + ((s0 - M.hA) & (MG_C - 1));
            len = e0 - s0;
          }
        }
      } else if (lane == 3 || lane == 4) {  // B' pieces
        const u64 lb = M.nb - M.hB;
        const u64 ye = j1 < lb ? j1 : lb;
        if (j0 < ye) {
          const u64 ce = ((j0 >> MG_LOGC) + 1) * MG_C;
          const u64 s0 = lane == 3 ? j0 : ce, e0 = lane == 3 ? (ce < ye ? ce : ye) : ye;
          if (s0 < e0) {
            ph = M.hA + ((u64)(lane == 3 ? db0 : db1) << MG_LOGC) + (s0 & (MG_C - 1));
            len = e0 - s0;
          }
        }
      } else if (lane == 5) {  // B tail
        const u64 lb = M.nb - M.hB;
        const u64 ys = j0 > lb ? j0 : lb;
        if (ys < j1) { ph = M.na + ys; len = j1 - ys; }
      }
      const u32 par = (u32)(((uintptr_t)(a + ph) >> 3) & 1u);
      const u32 bytes = len ? ((par + (u32)len) * 8u + 15u) & ~15u : 0u;
      u32 lo = (u32)len, bo = bytes;  // exclusive prefix sums over lanes 0..5
#pragma unroll
      for (int o = 1; o < 8; o <<= 1) {
        const u32 l2 = __shfl_up_sync(0xffffffffu, lo, o), b2 = __shfl_up_sync(0xffffffffu, bo, o);
        if (lane >= (u32)o) { lo += l2; bo += b2; }
      }
      const u32 total = __shfl_sync(0xffffffffu, bo, 7);
      lo -= (u32)len;
      bo -= bytes;
      if (lane < 6) {
        s_seg[sb][2 + lane] = len ? lo : 0xffffffffu;
        s_seg[sb][8 + lane] = bo / 8 + par;
      }
      if (lane == 0) {
        s_seg[sb][0] = (u32)(i1 - i0);
        s_seg[sb][1] = (u32)(j1 - j0);
      }
      __syncwarp();
      // the expect_tx arrive releases the map above to whoever observes the flip
      if (lane == 0) mbar_expect_tx(&s_full[sb], total);
      __syncwarp();
      if (lane < 6 && len) tma_load_1d(stage + bo / 8, a + ph - par, bytes, &s_full[sb]);
    };
    // every block <= upto has reported loaded (lanes poll 8 CTAs each).
    // WAR only: the store is issued after these loads returned the flags, and
    // a flag goes up only after its reader's bulk loads landed.
    constexpr int MAXS = 8;  // G <= 256
    auto wait_loaded = [&](u64 upto) -> bool {
      u64 spins = 0;
      for (;;) {
        bool ready = true;
#pragma unroll
        for (int q = 0; q < MAXS; ++q) {
          const u32 c = lane + 32 * q;
          if (c >= G || c > upto) continue;
          const u32 mc = c + (((u32)upto - c) / G) * G;  // 32-bit: NB < 2^32
          if (ld_relaxed_u32(M.status + c) < mc + 1) ready = false;
        }
        // WAR only: the store below is issued after these loads returned the
        // flags, and a flag goes up only after its reader's bulk loads landed
        if (__all_sync(0xffffffffu, ready)) return true;
        int ok = 1;
        if (lane == 0) {
          if (++spins > 32) __nanosleep(64);
          if ((spins & 1023) == 0) {
            if (ld_relaxed_u32(&g->sync.abort)) ok = 0;
            else if (spins > (1ull << 25)) { atomicExch(&g->sync.abort, 1u); ok = 0; }
          }
        }
        if (!__shfl_sync(0xffffffffu, ok, 0)) return false;
      }
    };
    fetch_plan(b);
    for (u64 j = 0; j < nblk && j < 2; ++j) issue_load(b + j * G, (int)j);
    // (an event loop that polls loads, refills and the dataflow rule without
    // blocking measured slower: 38 vs 32 ms at 2^32 — the status poll is an
    // L2 round trip on every pass)
    bool ok = true;
    bool owe_ofree = false;  // a store's read of s_obuf is still in flight
    auto settle_ofree = [&]() {
      if (owe_ofree && lane == 0) {
        bulk_wait_read_all();
        mbar_arrive(&s_ofree);
      }
      owe_ofree = false;
      __syncwarp();
    };
    for (u64 j = 0; j < nblk; ++j) {
      const u64 m = b + j * G;
      const int sb = (int)(j & 1);
      const u32 use = (u32)(j >> 1);
      if (j == 0) {  // publish block 0's load
        if (!wait_or_abort(&s_full[0], 0)) { ok = false; break; }
        if (lane == 0) st_relaxed_u32(M.status + b, (u32)(m + 1));
      }
      // the merge warps have read block j: its staging buffer takes block j+2
      if (!in_place(j)) {
        if (!wait_or_abort(&s_sfree[sb], use & 1)) { ok = false; break; }
        if (j + 2 < nblk) {
          if (lane == 0) fence_proxy_async_smem();
          __syncwarp();
          issue_load(m + 2 * G, sb);
        }
      }
      // the merge warps need s_obuf back before they can finish block j: the
      // previous store's read is waited for only now, not right after issue
      settle_ofree();
      // publish block j+1's load as soon as it has landed
      if (j + 1 < nblk) {
        if (!wait_or_abort(&s_full[sb ^ 1], ((j + 1) >> 1) & 1)) { ok = false; break; }
        if (lane == 0) st_relaxed_u32(M.status + b, (u32)(m + G + 1));
      }
      mark(0);
      if (!wait_or_abort(&s_ofull, (u32)(j & 1))) { ok = false; break; }  // output written
      mark(1);
      if (keep0 && j == 0) continue;  // block 0 is written after the final barrier
      const u64 upto = m + M.L < M.NB - 1 ? m + M.L : M.NB - 1;
      if (!(M.dbg & 1) && !wait_loaded(upto)) { ok = false; break; }
      mark(2);
      const u64* out = in_place(j) ? smem + sb * MG_STAGE_WORDS : s_obuf;
      if (lane == 0) {
        const u64 p0 = m * MG_C, p1 = (m + 1) * MG_C < M.n ? (m + 1) * MG_C : M.n;
        const u32 len = (u32)(p1 - p0);
        const u32 head = (u32)(((uintptr_t)(a + p0) >> 3) & 1u);
        const u32 body = len > head ? ((len - head) & ~1u) : 0u;
        if (head && len) a[p0] = out[0];
        if (head + body < len) a[p0 + len - 1] = out[len - 1];
        if (body) {
          tma_store_1d(a + p0 + head, out + head, body * 8u);
          bulk_commit();
        }
        if (in_place(j)) bulk_wait_read_all();  // the staging buffer is refilled below
      }
      owe_ofree = !in_place(j);  // settled (read waited, s_ofree arrived) next iteration
      __syncwarp();
      if (in_place(j) && j + 2 < nblk) {  // the store has read it: refill
        if (lane == 0) fence_proxy_async_smem();
        __syncwarp();
        issue_load(m + 2 * G, sb);
      }
      mark(3);
    }
    settle_ofree();
    if (lane == 0) bulk_wait_all();
    if (!ok && lane == 0) atomicExch(&g->sync.abort, 1u);
  } else {
    // ================================================= merge warps
    const u32 t = tid - 32;
    const u32 r0_all = (u32)(((u64)t * MG_C) / NMW), r1_all = (u32)(((u64)(t + 1) * MG_C) / NMW);
    u32 ofree_uses = 0;  // completed phases of s_ofree
    for (u64 j = 0; j < nblk; ++j) {
      const int sb = (int)(j & 1);
      if (!wait_or_abort(&s_full[sb], (u32)((j >> 1) & 1))) break;
      u64* sp = smem + sb * MG_STAGE_WORDS;
      const u32 na = s_seg[sb][0], nb = s_seg[sb][1], total = na + nb;
      const u32 r0 = r0_all < total ? r0_all : total, r1 = r1_all < total ? r1_all : total;
      // segment map: A side segments 0..2, B side 3..5 (lo = logical start,
      // 0xffffffff if absent); staging word = logical + offset of its segment
      const u32 la1 = s_seg[sb][3], la2 = s_seg[sb][4];
      const u32 oa0 = s_seg[sb][2] == 0xffffffffu ? 0u : s_seg[sb][8] - s_seg[sb][2];
      const u32 oa1 = s_seg[sb][9] - la1, oa2 = s_seg[sb][10] - la2;
      const u32 lb4 = s_seg[sb][6], lb5 = s_seg[sb][7];
      const u32 ob3 = s_seg[sb][5] == 0xffffffffu ? 0u : s_seg[sb][11] - s_seg[sb][5];
      const u32 ob4 = s_seg[sb][12] - lb4, ob5 = s_seg[sb][13] - lb5;
      auto mapA = [&](u32 x) -> u32 { return x + (x >= la2 ? oa2 : (x >= la1 ? oa1 : oa0)); };
      auto mapB = [&](u32 x) -> u32 { return x + (x >= lb5 ? ob5 : (x >= lb4 ? ob4 : ob3)); };
      u64 o[MO];
      if (r0 < r1) {
        u32 lo = r0 > nb ? r0 - nb : 0, hi = r0 < na ? r0 : na;
        while (lo < hi) {
          const u32 mid = (lo + hi) >> 1;
          if (sp[mapA(mid)] <= sp[mapB(na + r0 - mid - 1)]) lo = mid + 1;
          else hi = mid;
        }
        u32 i = lo, jj = r0 - lo;
        u64 ka = sp[mapA(i)];
        u64 kb = sp[mapB(na + jj)];
#pragma unroll
        for (int q = 0; q < MO; ++q) {
          const bool pa = (jj >= nb) || (i < na && ka <= kb);  // ties from A
          o[q] = pa ? ka : kb;
          const u32 ni = i + (pa ? 1u : 0u), nj = jj + (pa ? 0u : 1u);
          // unconditional load (one word past a side's end is still staging
          // memory), then select: no divergent branch per step
          const u64 nk = sp[pa ? mapA(ni) : mapB(na + nj)];
          ka = pa ? nk : ka;
          kb = pa ? kb : nk;
          i = ni;
          jj = nj;
        }
      }
      mark(0);
      named_bar(1, NMW);  // every merge warp is done reading the staging buffer
      u64* out = s_obuf;
      if (in_place(j)) {
        out = sp;
      } else {
        if (t == 0) mbar_arrive(&s_sfree[sb]);
        if (j > 0 && !(keep0)) {  // the previous block's store has read s_obuf
          if (!wait_or_abort(&s_ofree, ofree_uses & 1)) break;
          ++ofree_uses;
        }
      }
      mark(1);
#pragma unroll
      for (int q = 0; q < MO; ++q)
        if (r0 + q < r1) out[r0 + q] = o[q];
      fence_proxy_async_smem();
      named_bar(1, NMW);
      if (t == 0) mbar_arrive(&s_ofull);
      mark(2);
    }
  }
  if (prof && tid == 32)
    for (int q = 0; q < 3; ++q) g->sec[q] = cyc[q];
  if (prof && tid == 0) {
    g->sec[3] = cyc[0] + cyc[1];  // waiting for loads to land / for the merge warps
    g->sec[4] = cyc[2];           // dataflow rule
    g->sec[5] = cyc[3];           // store (+ refill issue)
  }
  if (M.hA > 0) {
    if (!grid_barrier(&g->sync, gen)) return;
    if (b == 0) {
      const u64 p1 = MG_C < M.n ? MG_C : M.n;
      for (u32 k = tid; k < (u32)p1; k += MG_THREADS) a[k] = s_obuf[k];
    }
  }
  if (tm) g->t[5] = globaltimer_ns();
}

// ---------------------------------------------------------------------------
// single-CTA merge of a small array (n <= C)
__global__ void __launch_bounds__(MG_THREADS, 1) merge_small_kernel(u64* a, u32 n, u32 na) {
  extern __shared__ __align__(16) u64 smem[];
  u64* s_in = smem;
  u64* s_out = smem + MG_IN_WORDS;
  for (u32 k = threadIdx.x; k < n; k += MG_THREADS) s_in[SI(k)] = a[k];
  __syncthreads();
  block_merge(s_in, na, n - na, s_out);
  __syncthreads();
  for (u32 k = threadIdx.x; k < n; k += MG_THREADS) a[k] = s_out[SO(k)];
}

// sortedness of both runs (debug=True): counts descents inside each run
__global__ void check_sorted_kernel(const u64* a, u64 n, u64 na, u32* bad) {
  const u64 stride = (u64)gridDim.x * blockDim.x;
  u32 c = 0;
  for (u64 k = (u64)blockIdx.x * blockDim.x + threadIdx.x; k + 1 < n; k += stride) {
    if (k + 1 == na) continue;  // run boundary
    c += a[k + 1] < a[k];
  }
  c = __reduce_add_sync(0xffffffffu, c);
  if ((threadIdx.x & 31) == 0 && c) atomicAdd(bad, c);
}

// ---------------------------------------------------------------------------
// host

struct MergeLayout {
  size_t dest, inv, lab0, lab1, jmp0, jmp1, visited, cr, plan, status, g, cut, total;
  u64 D, ncuts, desc_bytes;
};

// budget_words == 0: strong schedule, cut buffer of one chunk per SM
static MergeLayout merge_layout(u64 n, u64 na, u64 budget_words, int grid) {
  const u64 nb = n - na;
  const u64 hA = na % MG_C, hB = nb % MG_C;
  const u64 K = (n - hA - hB) / MG_C;
  const u64 NB = (n + MG_C - 1) / MG_C;
  MergeLayout L{};
  size_t off = 0;
  auto take = [&](size_t bytes) {
    size_t o = off;
    off += (bytes + 15) & ~(size_t)15;
    return o;
  };
  L.dest = take(K * 4);
  L.inv = take(K * 4);
  L.lab0 = take(K * 4);
  L.lab1 = take(K * 4);
  L.jmp0 = take(K * 4);
  L.jmp1 = take(K * 4);
  L.visited = take(K);
  L.cr = take((NB + 1) * 8);
  L.plan = take(NB * 32);
  L.status = take((size_t)grid * 4);
  L.g = take(sizeof(MergeGlobal));
  L.desc_bytes = off;
  const u64 desc_words = (off + 7) / 8;
  u64 cut_chunks;
  if (budget_words == 0) cut_chunks = (u64)grid;
  else cut_chunks = budget_words > desc_words ? (budget_words - desc_words) / MG_C : 0;
  if (cut_chunks > K) cut_chunks = K;
  if (cut_chunks) {
    L.D = (K + cut_chunks - 1) / cut_chunks;
    L.ncuts = (K + L.D - 1) / L.D;
  } else {
    L.D = 1;
    L.ncuts = 0;
  }
  L.cut = take(L.ncuts * MG_C * 8);
  L.total = off;
  return L;
}

static int merge_grid() { return num_sms(current_device()) * MG_CTAS_PER_SM; }

size_t merge_workspace_bytes(u64 n, u64 split, u64 budget_words) {
  if (split > n || n <= MG_C || split == 0 || split == n) return 0;
  return merge_layout(n, split, budget_words, merge_grid()).total;
}

int merge_device(u64* a, u64 n, u64 split, int check_sorted, void* ws, size_t ws_bytes,
                 void* scratch, size_t scratch_bytes, cudaStream_t st) {
  if (split > n) return PIP_ERR_INVALID_ARG;
  if (check_sorted && n > 1) {
    if (!scratch || scratch_bytes < 16) return PIP_ERR_OOM;
    u32* bad = (u32*)scratch;
    PIP_CUDA(cudaMemsetAsync(bad, 0, 4, st));
    u64 blocks = (n + 255) / 256;
    const u64 cap = (u64)num_sms(current_device()) * 8;
    if (blocks > cap) blocks = cap;
    check_sorted_kernel<<<(unsigned)blocks, 256, 0, st>>>(a, n, split, bad);
    PIP_CHECK_LAUNCH();
    u32 h = 0;
    PIP_CUDA(cudaMemcpyAsync(&h, bad, 4, cudaMemcpyDeviceToHost, st));
    PIP_CUDA(cudaStreamSynchronize(st));
    if (h) return PIP_ERR_UNSORTED;
  }
  if (n < 2 || split == 0 || split == n) return PIP_OK;
  if (n <= MG_C) {
    const size_t smem = (MG_IN_WORDS + MG_OUT_WORDS) * sizeof(u64);
    PIP_CUDA(cudaFuncSetAttribute(merge_small_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  (int)smem));
    merge_small_kernel<<<1, MG_THREADS, smem, st>>>(a, (u32)n, (u32)split);
    PIP_CHECK_LAUNCH();
    return PIP_OK;
  }
  const int grid = merge_grid();
  // the workspace the caller sized with pip_merge_workspace_bytes(n, split, b)
  // determines the cut buffer; recover b's layout from its size
  MergeLayout L = merge_layout(n, split, 0, grid);
  {
    const MergeLayout Lb = merge_layout(n, split, (u64)(ws_bytes / 8), grid);
    if (Lb.total <= ws_bytes) L = Lb;
    else {
      const MergeLayout L0 = merge_layout(n, split, 1, grid);  // descriptors only
      if (L0.total <= ws_bytes && L.total > ws_bytes) L = L0;
    }
  }
  if (!ws || ws_bytes < L.total) return PIP_ERR_OOM;
  if (((n + MG_C - 1) / MG_C) > 0xffffffffull) return PIP_ERR_UNSUPPORTED;
  char* w = (char*)ws;
  MergeArgs M{};
  {
    const char* e = getenv("PIP_MERGE_DBG");
    M.dbg = e ? (u32)atoi(e) : 0u;
  }
  M.a = a;
  M.n = n;
  M.na = split;
  M.nb = n - split;
  M.hA = split % MG_C;
  M.hB = M.nb % MG_C;
  M.KA = (split - M.hA) / MG_C;
  M.KB = (M.nb - M.hB) / MG_C;
  M.K = M.KA + M.KB;
  M.NB = (n + MG_C - 1) / MG_C;
  M.D = L.D;
  M.ncuts = L.ncuts;
  M.L = 1 + (M.hA + M.hB + MG_C - 1) / MG_C;
  M.cut = (u64*)(w + L.cut);
  M.dest = (u32*)(w + L.dest);
  M.inv = (u32*)(w + L.inv);
  M.lab[0] = (u32*)(w + L.lab0);
  M.lab[1] = (u32*)(w + L.lab1);
  M.jmp[0] = (u32*)(w + L.jmp0);
  M.jmp[1] = (u32*)(w + L.jmp1);
  M.visited = (unsigned char*)(w + L.visited);
  M.cr = (u64*)(w + L.cr);
  M.plan = (ulonglong4*)(w + L.plan);
  M.status = (u32*)(w + L.status);
  M.g = (MergeGlobal*)(w + L.g);
  if ((u64)grid <= 2 * M.L || grid > 256) return PIP_ERR_UNSUPPORTED;
  PIP_CUDA(cudaMemsetAsync(M.status, 0, (size_t)grid * 4, st));
  PIP_CUDA(cudaMemsetAsync(M.g, 0, sizeof(MergeGlobal), st));
  const size_t smem = MG_SMEM;
  PIP_CUDA(cudaFuncSetAttribute(merge_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  void* args[] = {&M};
  PIP_CUDA(cudaLaunchCooperativeKernel((const void*)merge_kernel, dim3(grid), dim3(MG_THREADS), args,
                                       smem, st));
  MergeGlobal gh{};
  PIP_CUDA(cudaMemcpyAsync(&gh, M.g, sizeof(gh), cudaMemcpyDeviceToHost, st));
  PIP_CUDA(cudaStreamSynchronize(st));
  if (gh.sync.abort) return PIP_ERR_CUDA;
  if (timing_enabled() && (M.dbg & 4))
    fprintf(stderr, "[pip merge] CTA0 cycles: merge warps: merge (+ wait data) %llu | wait output buffer %llu | write-out %llu ; "
            "control: loads/merge wait %llu | dataflow wait %llu | store %llu\n",
            (unsigned long long)gh.sec[0], (unsigned long long)gh.sec[1], (unsigned long long)gh.sec[2],
            (unsigned long long)gh.sec[3], (unsigned long long)gh.sec[4], (unsigned long long)gh.sec[5]);
  if (timing_enabled())
    fprintf(stderr,
            "[pip merge] n=%llu K=%llu ncuts=%llu D=%llu uncut=%u  P0 %.3f ms | cuts %.3f | "
            "walks %.3f | uncut %.3f | block-merge %.3f ms\n",
            (unsigned long long)n, (unsigned long long)M.K, (unsigned long long)M.ncuts,
            (unsigned long long)M.D, gh.uncut, (gh.t[1] - gh.t[0]) * 1e-6,
            (gh.t[2] - gh.t[1]) * 1e-6, (gh.t[3] - gh.t[2]) * 1e-6, (gh.t[4] - gh.t[3]) * 1e-6,
            (gh.t[5] - gh.t[4]) * 1e-6);
  return PIP_OK;
}

}  // namespace pip
