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

static constexpr int MG_THREADS = 544;  // block phase: loader + watcher + 15 merge warps
static constexpr int MG_CP = 512;       // threads that move chunks (P1) / small merges
static constexpr int MG_CTAS_PER_SM = 1;
static constexpr u32 MG_LOGC = 13;
static constexpr u64 MG_C = 1ull << MG_LOGC;  // words per chunk / output block
static constexpr int MG_PER_THREAD = (int)(MG_C / MG_CP);
// shared-memory padding: merge-path readers sit ~8 words apart and writers
// exactly 16 words apart, which on 8-byte words means 16- and 32-way bank
// conflicts; one pad word per 8 (inputs) / per 16 (outputs) spreads them
__device__ __forceinline__ u32 SI(u32 l) { return l + (l >> 3); }
__device__ __forceinline__ u32 SO(u32 r) { return r + (r >> 4); }
static constexpr u32 MG_IN_WORDS = (u32)(MG_C + MG_C / 8);
static constexpr u32 MG_OUT_WORDS = (u32)(MG_C + MG_C / 16);
static constexpr u32 MG_STAGE_WORDS = (u32)(MG_C + 16);  // bulk-copy staging (+2 junk words x 6 segments)
// per merge warp: a transpose tile for its <= 32 * 8192 / 480 + 1 outputs
static constexpr u32 MG_SCR = (u32)((32 * MG_C) / (MG_THREADS - 64) + 4);
// per-CTA load status words one L2 line apart: every CTA polls its
// neighbours' words, and packed words made a few lines a hot spot
static constexpr u32 MG_SST = 32;
// at most this many slots on cut-free cycles: one CTA rotates them serially
static constexpr u32 MG_UNCUT_SERIAL = 2048;
static constexpr size_t MG_SMEM = (size_t)(2 * MG_STAGE_WORDS + (MG_THREADS / 32 - 2) * MG_SCR) * 8;

struct MergeGlobal {
  GridSync sync;
  u32 walk_next;  // dynamic walk assignment
  u32 uncut;      // #slots on cut-free cycles
  u64 t[8];       // %globaltimer at phase boundaries (CTA 0)
  u64 sec[8];     // PIP_MERGE_DBG bit2: CTA 0 cycles (merge warps: data wait|merge|ofree wait|write-out; control: loads|dataflow|store)
};

struct MergeArgs {
  u32 dbg;  // PIP_MERGE_DBG: bit0 skip the dataflow wait (profiling), bit1 no merge (profiling), bit2 CTA 0 cycle counters,
            // bit3 mapped staging, bit4 global dataflow rule, bit5 pointer jumping for cut-free cycles (tests),
            // bit6 8-byte write-out stores, bit8 bisect the whole diagonal (no gallop),
            // bit9 16-byte LSU write-out stores instead of one bulk copy per warp
  u64* a;
  u64 n, na, nb;
  u64 hA, hB, KA, KB, K, NB, D, ncuts, L;
  u64* cut;       // [ncuts * C] saved chunks of the cut slots
  u32* dest;      // [K] destination slot of the chunk in slot s
  u32* inv;       // [K] slot whose chunk moves into slot s
  u32* lab[2];    // [K] pointer-jumping labels   (only if uncut cycles)
  u32* jmp[2];    // [K] pointer-jumping jumps
  unsigned char* visited;  // [K]
  u32* rlo;       // [K] first / last output block that reads the chunk in slot s
  u32* rhi;       //     (after the permutation); rlo = ~0 if none
  u64* cr;        // [NB + 1] A co-rank of every output block boundary
  ulonglong4* plan;  // [NB] {i0, i1, dest slots of the <= 2 A' and <= 2 B' chunks}
  u32* status;    // [G * MG_SST] per CTA: (last block loaded) + 1
  u64* head_save; // [C] block 0's output while the in-place head may still be read
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

// smallest i in [lo, hi] with !pred(i), pred monotone (true, then false):
// gallop from the estimate g in steps st, 2st, ..., then bisect the bracket
// (random probes go to HBM in P0: a close estimate saves most of them)
template <class P>
__device__ __forceinline__ u64 gallop_lb(u64 lo, u64 hi, u64 g, u64 st, P pred) {
  if (lo < hi) {
    g = g < lo ? lo : (g >= hi ? hi - 1 : g);
    if (pred(g)) {
      lo = g + 1;
      for (; lo + st <= hi; st <<= 1) {
        if (pred(lo + st - 1)) lo += st;
        else { hi = lo + st - 1; break; }
      }
    } else {
      hi = g;
      for (; hi >= lo + st; st <<= 1) {
        if (!pred(hi - st)) hi -= st;
        else { lo = hi - st + 1; break; }
      }
    }
  }
  while (lo < hi) {
    const u64 mid = (lo + hi) >> 1;
    if (pred(mid)) lo = mid + 1; else hi = mid;
  }
  return lo;
}

// merge path over the original runs A = a[0:na), B = a[na:n) (A first on ties)
__device__ __forceinline__ u64 corank2_global(const MergeArgs& M, u64 q) {
  const u64* A = M.a;
  const u64* B = M.a + M.na;
  const u64 lo0 = q > M.nb ? q - M.nb : 0, hi0 = q < M.na ? q : M.na;
  if (!(M.dbg & 256))
    return gallop_lb(lo0, hi0, (u64)(((unsigned __int128)q * M.na) / M.n), 64,
                     [&](u64 i) { return __ldcg(A + i) <= __ldcg(B + (q - i - 1)); });
  u64 lo = lo0, hi = hi0;
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
  if (tid < MG_CP) {
#pragma unroll
    for (int k = 0; k < MG_PER_THREAD; ++k) v[k] = __ldcg(src + tid + k * MG_CP);
  }
  __syncthreads();
  if (tid < MG_CP) {
#pragma unroll
    for (int k = 0; k < MG_PER_THREAD; ++k) dst[tid + k * MG_CP] = v[k];
  }
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
        // #B' chunks with last < this last (estimate: proportional position)
        const u64 c = gallop_lb(0, M.KB, (u64)(((unsigned __int128)x * M.KB) / (M.KA ? M.KA : 1)), 4,
                                [&](u64 mid) { return __ldcg(a + M.na + ((mid + 1) << MG_LOGC) - 1) < last; });
        d = x + c;
      } else {
        const u64 y = x - M.KA;
        const u64 last = __ldcg(a + M.na + ((y + 1) << MG_LOGC) - 1);
        // #A' chunks with last <= this last
        const u64 c = gallop_lb(0, M.KA, (u64)(((unsigned __int128)y * M.KA) / (M.KB ? M.KB : 1)), 4,
                                [&](u64 mid) { return __ldcg(a + M.hA + ((mid + 1) << MG_LOGC) - 1) <= last; });
        d = y + c;
      }
      M.dest[x] = (u32)d;
      M.inv[d] = (u32)x;
      M.visited[x] = 0;
      M.rlo[x] = 0xffffffffu;
      M.rhi[x] = 0;
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
      // reader ranges of the slots this block loads from (the rule in P2)
      if (xs < i1) {
        atomicMin(M.rlo + da0, (u32)m); atomicMax(M.rhi + da0, (u32)m);
        atomicMin(M.rlo + da1, (u32)m); atomicMax(M.rhi + da1, (u32)m);
      }
      if (j0 < ye) {
        atomicMin(M.rlo + db0, (u32)m); atomicMax(M.rhi + db0, (u32)m);
        atomicMin(M.rlo + db1, (u32)m); atomicMax(M.rhi + db1, (u32)m);
      }
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
    // count the slots on cut-free cycles and list them (warp-aggregated
    // appends into the pointer-jumping array, unused by the serial path)
    const u64 cap = M.K < MG_UNCUT_SERIAL ? M.K : MG_UNCUT_SERIAL;
    const u32 lane = tid & 31;
    for (u64 x0 = s; x0 < e; x0 += MG_THREADS) {
      const u64 x = x0 + tid;
      const bool cand = x < e && !__ldcg(M.visited + x) && __ldcg(M.inv + x) != (u32)x;
      const unsigned bal = __ballot_sync(0xffffffffu, cand);
      if (!bal) continue;
      u32 base = 0;
      if (lane == 0) base = atomicAdd(&g->uncut, (u32)__popc(bal));
      base = __shfl_sync(0xffffffffu, base, 0);
      const u64 idx = base + (u32)__popc(bal & ((1u << lane) - 1u));
      if (cand && idx < cap) M.lab[0][idx] = (u32)x;
    }
  }
  if (!grid_barrier(&g->sync, gen)) return;
  const u32 n_uncut = ld_relaxed_u32(&g->uncut);
  if (n_uncut && n_uncut <= MG_UNCUT_SERIAL && !(M.dbg & 32)) {
    // few slots (the usual case with a cut buffer): CTA 0 rotates each cycle
    // of the listed slots through shared memory — no pointer-jumping rounds
    if (b == 0) {
      const u32 cnt = n_uncut;  // <= min(K, MG_UNCUT_SERIAL): all listed in P1b
      for (u32 c = 0; c < cnt; ++c) {
        const u64 x0 = __ldcg(M.lab[0] + c);
        // thread 0 alone reads and writes `visited` here (program order)
        if (tid == 0) s_flag = !__ldcg(M.visited + x0);
        __syncthreads();
        const bool lead = s_flag != 0;
        __syncthreads();
        if (!lead) continue;
        for (u32 k = tid; k < MG_C; k += MG_THREADS) s_out[k] = __ldcg(slot_ptr(M, x0) + k);
        __syncthreads();
        u64 sdst = x0;
        for (u64 steps = 0; steps <= M.K; ++steps) {
          if (tid == 0) M.visited[sdst] = 1;
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
    }
    if (!grid_barrier(&g->sync, gen)) return;
  } else if (n_uncut) {
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
  // Warp-specialized: warp 0 loads, warp 1 watches the dataflow rule, warps
  // 2..16 merge and store.
  //   load   (control) the <= 6 contiguous input segments of a block (A head
  //          in place, <= 2 permuted A' chunks, <= 2 permuted B' chunks, B
  //          tail in place), one bulk copy each into one of two staging
  //          buffers (widened to 16-byte alignment); "loaded" is published as
  //          soon as the bytes land;
  //   rule   (watcher) block m may be written once every block <= m + L has
  //          loaded: polled ahead of the merge warps, announced to them
  //          through a monotone shared counter;
  //   merge  (merge warps) a merge-path range of 17-18 consecutive outputs per
  //          thread into registers, straight from staging (each side one
  //          contiguous range when the chunk grid is 16-byte aligned, else
  //          through a segment map); every warp hands the staging buffer back
  //          on its own (mbarrier, 15 arrivals) — no CTA-wide barrier;
  //   store  (merge warps) each warp transposes its ~546 outputs through a
  //          private shared-memory tile and writes them with coalesced
  //          stores once the rule allows: no output buffer shared by the
  //          CTA, so no block waits for the previous block's store.
  constexpr u32 NMW = MG_THREADS - 64;  // merge threads
  constexpr int MO = (int)((MG_C + NMW - 1) / NMW) + 1;  // outputs per thread, at most
  u64* s_scr = smem + 2 * MG_STAGE_WORDS;  // per merge warp: MG_SCR words
  __shared__ __align__(8) u64 s_full[2], s_sfree[2];
  __shared__ u32 s_seg[2][2 + 2 * 6];  // per buffer: na, nb | lo[6] | staging index[6]
  __shared__ u32 s_dfdone;  // blocks (of this CTA) whose dataflow rule holds
  // CTA 0 writes block 0 (it overwrites the in-place head, which any block
  // may still read) to M.head_save; it is copied home after a final barrier
  const bool keep0 = M.hA > 0 && b == 0;
  // interior piece boundaries of every block sit at a + hA + s*C (chunk
  // starts, hA, the tail start): contiguous staging iff that is 16-byte aligned
  const bool contig = ((((uintptr_t)(a + M.hA)) >> 3) & 1u) == 0 && !(M.dbg & 8);
  const u64 nblk = b < M.NB ? (M.NB - 1 - b) / G + 1 : 0;  // blocks of this CTA
  auto wait_or_abort = [&](u64* bar, u32 ph) -> bool {
    u32 n = 0;
    while (!mbar_try(bar, ph))
      if ((++n & 255) == 0 && ld_relaxed_u32(&g->sync.abort)) return false;
    return true;
  };
  if (tid == 0) {
    for (int q = 0; q < 2; ++q) {
      mbar_init(&s_full[q], 1);
      mbar_init(&s_sfree[q], NMW / 32);
    }
    s_dfdone = 0;
    mbar_fence_init();
  }
  __syncthreads();

  const bool prof = (M.dbg & 4) && b == 0 && (tid == 0 || (tid >= 32 && tid < 64) || tid == 64);
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
      lo -= (u32)len;
      bo -= bytes;
      u32 total;
      if (contig) {
        // every piece after the first of its side starts (and the one before
        // it ends) 16-byte aligned, so each side is one contiguous range of
        // staging: A at sA = parity of its first word, B from the next even
        // word after A (+ its first word's parity); copies never overlap
        const u32 na_b = (u32)(i1 - i0);
        const unsigned pres = __ballot_sync(0xffffffffu, lane < 6 && len != 0);
        const unsigned presA = pres & 7u, presB = pres & 0x38u;
        const u32 parA = presA ? (u32)__shfl_sync(0xffffffffu, par, __ffs(presA) - 1) : 0u;
        const u32 parB = presB ? (u32)__shfl_sync(0xffffffffu, par, __ffs(presB) - 1) : 0u;
        const u32 sA = parA, sB = ((sA + na_b + 1u) & ~1u) + parB;
        const u32 st = lane < 3 ? sA + lo : sB + (lo - na_b);  // staging word of this piece
        bo = (st - par) * 8u;
        total = __reduce_add_sync(0xffffffffu, lane < 6 ? bytes : 0u);
        if (lane == 0) {
          s_seg[sb][2] = sA;
          s_seg[sb][3] = sB;
        }
      } else {
        total = __shfl_sync(0xffffffffu, bo + bytes, 7);
        if (lane < 6) {
          s_seg[sb][2 + lane] = len ? lo : 0xffffffffu;
          s_seg[sb][8 + lane] = bo / 8 + par;
        }
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
    fetch_plan(b);
    for (u64 j = 0; j < nblk && j < 2; ++j) issue_load(b + j * G, (int)j);
    bool ok = true;
    for (u64 j = 0; j < nblk && ok; ++j) {
      const u64 m = b + j * G;
      const int sb = (int)(j & 1);
      const u32 use = (u32)(j >> 1);
      if (j == 0) {  // publish block 0's load
        if (!wait_or_abort(&s_full[0], 0)) { ok = false; break; }
        if (lane == 0) st_relaxed_u32(M.status + MG_SST * b, (u32)(m + 1));
      }
      // two local events, whichever comes first: the merge warps have read
      // block j (its staging buffer takes block j+2) / block j+1 has landed
      // (publish it for the other CTAs' dataflow rule)
      bool iss = true, pub = j + 1 < nblk;
      u32 spins = 0;
      while (iss || pub) {
        if (iss && __shfl_sync(0xffffffffu, (int)mbar_try(&s_sfree[sb], use & 1), 0)) {
          iss = false;
          if (j + 2 < nblk) {
            if (lane == 0) fence_proxy_async_smem();
            __syncwarp();
            issue_load(m + 2 * G, sb);
          }
          mark(0);
        }
        if (pub && __shfl_sync(0xffffffffu, (int)mbar_try(&s_full[sb ^ 1], ((j + 1) >> 1) & 1), 0)) {
          pub = false;
          if (lane == 0) st_relaxed_u32(M.status + MG_SST * b, (u32)(m + G + 1));
          mark(1);
        }
        if ((++spins & 255) == 0 && ld_relaxed_u32(&g->sync.abort)) { ok = false; break; }
      }
    }
    if (!ok && lane == 0) atomicExch(&g->sync.abort, 1u);
  } else if (tid < 64) {
    // ================================================= dataflow watcher
    const u32 lane = tid & 31;
    // every block <= upto has reported loaded (lanes poll 8 CTAs each).
    // WAR only: the merge warps store after these loads returned the flags,
    // and a flag goes up only after its reader's bulk loads landed.
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
          if (ld_relaxed_u32(M.status + MG_SST * c) < mc + 1) ready = false;
        }
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
    // the precise form of the rule: block m overwrites (parts of) slots
    // q_lo..q_hi, whose chunks are read by the blocks rlo..rhi (computed in
    // P0b; rhi <= m + L) — only those must have loaded.  Blocks over the tail
    // use the global form (every block <= m + L).  Lane k watches block
    // jb + k of a 32-block window: one round of status loads checks all 32,
    // and the announced count is the prefix of satisfied blocks — the
    // watcher is not a chain of dependent L2 round trips per block.
    const u64 tail_blk = M.hB ? (M.n - M.hB) / MG_C : M.NB;  // first block over the tail
    bool ok = true;
    for (u64 jb = 0; jb < nblk && ok; jb += 32) {
      const u64 j = jb + lane;
      const u64 m = b + j * G;
      int mode = 0;  // 0 nothing to wait for, 1 blocks lo..hi, 2 every block <= hi
      u32 lo = 1, hi = 0;
      if (j < nblk && !(keep0 && j == 0) && !(M.dbg & 1)) {
        if (m >= tail_blk || (M.dbg & 16)) {
          mode = 2;
          hi = (u32)(m + M.L < M.NB - 1 ? m + M.L : M.NB - 1);
        } else {
          const u64 p0 = m * MG_C;
          const u64 qlo = p0 >= M.hA ? (p0 - M.hA) >> MG_LOGC : 0;
          const u64 qe = (p0 + MG_C - 1 >= M.hA ? ((p0 + MG_C - 1 - M.hA) >> MG_LOGC) : 0);
          const u64 qhi = qe < M.K - 1 ? qe : M.K - 1;
          lo = 0xffffffffu;
          for (u64 q = qlo; q <= qhi && q < M.K; ++q) {
            const u32 l1 = __ldcg(M.rlo + q), h1 = __ldcg(M.rhi + q);
            if (l1 <= h1) {  // the chunk in slot q has readers
              lo = l1 < lo ? l1 : lo;
              hi = h1 > hi ? h1 : hi;
            }
          }
          if (lo <= hi) mode = ((u64)hi - lo + 1 >= G) ? 2 : 1;
        }
      }
      bool sat = mode == 0;
      u64 spins = 0;
      for (;;) {
        // only the first few unsatisfied blocks of the window poll
        const unsigned bal0 = __ballot_sync(0xffffffffu, sat);
        const u32 k0 = bal0 == 0xffffffffu ? 32u : (u32)(__ffs(~bal0) - 1);
        if (!sat && mode == 1 && lane < k0 + 2) {
          // up to 4 readers with independent loads in flight (one round trip)
          u32 v[4];
#pragma unroll
          for (int q = 0; q < 4; ++q) {
            const u32 x = lo + q <= hi ? lo + q : hi;
            v[q] = ld_relaxed_u32(M.status + MG_SST * (x % G));
          }
          bool r = true;
#pragma unroll
          for (int q = 0; q < 4; ++q) {
            const u32 x = lo + q <= hi ? lo + q : hi;
            if (v[q] < x + 1u) r = false;
          }
          for (u32 x = lo + 4; x <= hi; ++x)
            if (ld_relaxed_u32(M.status + MG_SST * (x % G)) < x + 1u) r = false;
          if (prof && !r && lane == 0) cyc[4] += 1;  // unsatisfied polls of the window's first block
          sat = r;
        }
        if (prof && lane == 0) cyc[5] += 1;
        const unsigned bal = __ballot_sync(0xffffffffu, sat);
        const u32 k = bal == 0xffffffffu ? 32u : (u32)(__ffs(~bal) - 1);
        if (k > 0 && lane == 0) {
          __threadfence_block();
          *(volatile u32*)&s_dfdone = (u32)(jb + k);
        }
        if (k == 32) break;
        if (__shfl_sync(0xffffffffu, mode, k) == 2) {  // cooperative global wait
          const u32 upto = __shfl_sync(0xffffffffu, hi, k);
          if (!wait_loaded(upto)) { ok = false; break; }
          if (lane == k) sat = true;
          continue;
        }
        int go = 1;
        if (lane == 0) {
          if (++spins > 4) __nanosleep(128);
          if ((spins & 1023) == 0) {
            if (ld_relaxed_u32(&g->sync.abort)) go = 0;
            else if (spins > (1ull << 25)) { atomicExch(&g->sync.abort, 1u); go = 0; }
          }
        }
        if (!__shfl_sync(0xffffffffu, go, 0)) { ok = false; break; }
      }
      mark(2);
    }
    if (!ok && lane == 0) atomicExch(&g->sync.abort, 1u);
  } else {
    // ================================================= merge warps
    const u32 t = tid - 64, w = t >> 5, lane = t & 31;
    const u32 r0_all = (u32)(((u64)t * MG_C) / NMW), r1_all = (u32)(((u64)(t + 1) * MG_C) / NMW);
    const u32 wr0 = (u32)(((u64)(w * 32) * MG_C) / NMW), wr1 = (u32)(((u64)(w * 32 + 32) * MG_C) / NMW);
    bool bulk_pending = false;  // this warp's last bulk store may still read its tile
    for (u64 j = 0; j < nblk; ++j) {
      const u64 m = b + j * G;
      const int sb = (int)(j & 1);
      if (!wait_or_abort(&s_full[sb], (u32)((j >> 1) & 1))) break;
      mark(3);
      u64* sp = smem + sb * MG_STAGE_WORDS;
      const u32 na = s_seg[sb][0], nb = s_seg[sb][1], total = na + nb;
      const u32 r0 = r0_all < total ? r0_all : total, r1 = r1_all < total ? r1_all : total;
      u64 o[MO];
      if (M.dbg & 2) {  // profiling: no merge (outputs are garbage)
#pragma unroll
        for (int q = 0; q < MO; ++q) o[q] = sp[(r0 + q) & (MG_C - 1)];
      } else if (contig) {
        const u32 sA = s_seg[sb][2], sB = s_seg[sb][3];
        if (r0 < r1) {
          u32 lo = r0 > nb ? r0 - nb : 0, hi = r0 < na ? r0 : na;
          const u32 bq = sB + r0 - 1;  // B word of merge-path step mid: bq - mid
          // gallop from the proportional estimate r0 * na / total (the
          // co-rank of interleaved runs sits within a few tens of it), then
          // bisect the bracket: fewer dependent shared loads than bisecting
          // the whole diagonal; any input stays correct (brackets only grow)
          if (lo < hi && !(M.dbg & 256)) {
            u32 g = (u32)(((u64)r0 * na) / (total ? total : 1u));
            g = g < lo ? lo : (g >= hi ? hi - 1 : g);
            if (sp[sA + g] <= sp[bq - g]) {  // co-rank in (g, hi]
              lo = g + 1;
              for (u32 st = 16; lo + st <= hi; st <<= 1) {
                const u32 j = lo + st - 1;
                if (sp[sA + j] <= sp[bq - j]) lo = j + 1;
                else { hi = j; break; }
              }
            } else {  // co-rank in [lo, g]
              hi = g;
              for (u32 st = 16; hi >= lo + st; st <<= 1) {
                const u32 j = hi - st;
                if (!(sp[sA + j] <= sp[bq - j])) hi = j;
                else { lo = j + 1; break; }
              }
            }
          }
          while (lo < hi) {
            const u32 mid = (lo + hi) >> 1;
            if (sp[sA + mid] <= sp[bq - mid]) lo = mid + 1;
            else hi = mid;
          }
          // absolute staging indices; the word one past either side's end is
          // still staging memory, so the next-key load is unconditional
          u32 ai = sA + lo, bi = sB + (r0 - lo);
          const u32 ae = sA + na, be = sB + nb;
          u64 ka = sp[ai], kb = sp[bi];
          // (a second, bounds-free copy of this loop for threads whose range
          // cannot exhaust a side measured slower: 16.0 vs 14.0 ms at 2^32)
          {
#pragma unroll
            for (int q = 0; q < MO; ++q) {
              const bool pa = (bi >= be) || (ai < ae && ka <= kb);  // ties from A
              o[q] = pa ? ka : kb;
              ai += pa ? 1u : 0u;
              bi += pa ? 0u : 1u;
              const u64 nk = sp[pa ? ai : bi];
              ka = pa ? nk : ka;
              kb = pa ? kb : nk;
            }
          }
        }
      } else {
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
      }
      mark(0);
      // this warp is done with the staging buffer
      __syncwarp();
      if (lane == 0) mbar_arrive(&s_sfree[sb]);
      // the dataflow rule (announced by the watcher warp)
      {
        // sleep between polls: 15 spinning warps would take the issue slots
        // and the shared-memory pipe the loader and the watcher need
        u32 n = 0;
        while (*(volatile u32*)&s_dfdone < (u32)(j + 1)) {
          __nanosleep(128);
          if ((++n & 255) == 0 && ld_relaxed_u32(&g->sync.abort)) break;
        }
        __threadfence_block();
      }
      mark(1);
      // transpose through the warp's tile (placed at the 16-byte parity of
      // the destination), then coalesced 16-byte stores
      u64* gd = ((keep0 && j == 0) ? M.head_save : a + m * MG_C) + wr0;
      const u32 head = (u32)(((uintptr_t)gd >> 3) & 1u);
      u64* scr = s_scr + w * MG_SCR + head - wr0;  // indexed by block-relative rank
      // the tile may still be read by this warp's previous bulk store
      if (bulk_pending) {
        if (lane == 0) bulk_wait_read_all();
        __syncwarp();
        bulk_pending = false;
      }
#pragma unroll
      for (int q = 0; q < MO; ++q)
        if (r0 + q < r1) scr[r0 + q] = o[q];
      const u32 cnt = (wr1 < total ? wr1 : total) - (wr0 < total ? wr0 : total);
      const u64* sw = scr + wr0;  // sw[k] = output word gd[k]; gd + k, sw + k 16-byte aligned iff k = head mod 2
      if (!(M.dbg & (64 | 512))) {
        // one bulk copy per warp (the LSU issues no global stores); the
        // ragged first / last word by hand
        fence_proxy_async_smem();
        __syncwarp();
        if (lane == 0 && cnt) {
          const u32 body = (cnt - head) & ~1u;
          if (head) __stcs(gd, sw[0]);
          if (head + body < cnt) __stcs(gd + cnt - 1, sw[cnt - 1]);
          if (body) {
            tma_store_1d(gd + head, sw + head, body * 8u);
            bulk_commit();
          }
        }
        bulk_pending = true;
      } else if (M.dbg & 64) {
        __syncwarp();
        for (u32 k = lane; k < cnt; k += 32) gd[k] = sw[k];
      } else {
        __syncwarp();
        for (u32 k = head + 2 * lane; k + 1 < cnt; k += 64)
          __stcs(reinterpret_cast<ulonglong2*>(gd + k), *reinterpret_cast<const ulonglong2*>(sw + k));
        if (lane == 0 && cnt) {
          if (head) __stcs(gd, sw[0]);
          if (((cnt - head) & 1u) && cnt - 1 >= head) __stcs(gd + cnt - 1, sw[cnt - 1]);
        }
      }
      __syncwarp();
      mark(2);
    }
    if (lane == 0) bulk_wait_all();  // the stores have landed (head_save is read below)
    __syncwarp();
  }
  if (prof && tid == 64) {
    g->sec[0] = cyc[3];  // waiting for the block's loads to land
    for (int q = 0; q < 3; ++q) g->sec[1 + q] = cyc[q];
  }
  if (prof && tid == 0) g->sec[4] = cyc[0] + cyc[1];  // loader: refills + publishes
  if (prof && tid == 32) g->sec[5] = cyc[2];          // watcher: dataflow rule
  if ((M.dbg & 4) && b == 0 && tid < 64 && tid >= 32) {  // watcher lanes: missing-reader polls
    atomicAdd((unsigned long long*)&g->sec[6], (unsigned long long)cyc[4]);
    atomicAdd((unsigned long long*)&g->sec[7], (unsigned long long)cyc[5]);  // polls
  }
  if (M.hA > 0) {
    if (!grid_barrier(&g->sync, gen)) return;
    if (b == 0) {
      const u64 p1 = MG_C < M.n ? MG_C : M.n;
      for (u32 k = tid; k < (u32)p1; k += MG_THREADS) a[k] = __ldcg(M.head_save + k);
    }
  }
  if (tm) g->t[5] = globaltimer_ns();
}

// ---------------------------------------------------------------------------
// single-CTA merge of a small array (n <= C)
__global__ void __launch_bounds__(MG_CP, 1) merge_small_kernel(u64* a, u32 n, u32 na) {
  extern __shared__ __align__(16) u64 smem[];
  u64* s_in = smem;
  u64* s_out = smem + MG_IN_WORDS;
  for (u32 k = threadIdx.x; k < n; k += MG_CP) s_in[SI(k)] = a[k];
  __syncthreads();
  block_merge(s_in, na, n - na, s_out);
  __syncthreads();
  for (u32 k = threadIdx.x; k < n; k += MG_CP) a[k] = s_out[SO(k)];
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
  size_t dest, inv, lab0, lab1, jmp0, jmp1, visited, rlo, rhi, cr, plan, head, g, cut, total;
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
  L.rlo = take(K * 4);
  L.rhi = take(K * 4);
  L.cr = take((NB + 1) * 8);
  L.plan = take(NB * 32);
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
  // block 0's deferred output (only if there is an in-place head): the cut
  // buffer or the pointer-jumping arrays are dead by the block phase; only a
  // small array with a budget below one chunk needs C words of its own
  if (hA == 0 || L.ncuts > 0) L.head = L.cut;
  else if (L.visited - L.lab0 >= MG_C * 8) L.head = L.lab0;
  else L.head = take(MG_C * 8);
  L.total = off;
  return L;
}

// ---------------------------------------------------------------------------
// Streaming host merge (pip_merge_u64_host): the runs arrive over PCIe, so
// the device merges each output chunk out of place from the uploaded runs
// into a ring buffer that is copied straight back.  Chunk co-ranks come from
// the host (all computed before anything is written back), so a chunk only
// ever reads the part of the runs that has been uploaded.
//
// merge_copy_kernel: out[0 : na+nb) = merge(a[0:na), b[0:nb)), equal keys
// from a first (the co-rank rule of strong.py:474-488); one CTA per
// MC_TILE outputs, runs staged in shared memory, MC_ITEMS outputs per thread.
static constexpr int MC_THREADS = 256, MC_ITEMS = 8, MC_TILE = MC_THREADS * MC_ITEMS;

__device__ __forceinline__ u64 mc_corank(const u64* a, u64 na, const u64* b, u64 nb, u64 r) {
  u64 lo = r > nb ? r - nb : 0, hi = r < na ? r : na;
  while (lo < hi) {  // smallest i with not (b[r-i-1] >= a[i])
    const u64 mid = (lo + hi) >> 1;
    if (b[r - mid - 1] >= a[mid]) lo = mid + 1;
    else hi = mid;
  }
  return lo;
}

__global__ void __launch_bounds__(MC_THREADS)
merge_copy_kernel(const u64* __restrict__ a, u64 na, const u64* __restrict__ b, u64 nb,
                  u64* __restrict__ out) {
  __shared__ u64 s[MC_TILE + 1];
  __shared__ u64 s_i[2];
  const u64 n = na + nb;
  const u64 r0 = (u64)blockIdx.x * MC_TILE;
  const u64 r1 = r0 + MC_TILE < n ? r0 + MC_TILE : n;
  if (threadIdx.x == 0) s_i[0] = mc_corank(a, na, b, nb, r0);
  if (threadIdx.x == 32) s_i[1] = mc_corank(a, na, b, nb, r1);
  __syncthreads();
  const u64 i0 = s_i[0], i1 = s_i[1], j0 = r0 - i0;
  const u32 la = (u32)(i1 - i0), len = (u32)(r1 - r0), lb = len - la;
  for (u32 t = threadIdx.x; t < la; t += MC_THREADS) s[t] = a[i0 + t];
  for (u32 t = threadIdx.x; t < lb; t += MC_THREADS) s[la + t] = b[j0 + t];
  __syncthreads();
  const u32 q0 = threadIdx.x * MC_ITEMS;
  u64 v[MC_ITEMS];
  if (q0 < len) {
    u32 lo = q0 > lb ? q0 - lb : 0, hi = q0 < la ? q0 : la;
    while (lo < hi) {
      const u32 mid = (lo + hi) >> 1;
      if (s[la + q0 - mid - 1] >= s[mid]) lo = mid + 1;
      else hi = mid;
    }
    u32 ia = lo, ib = q0 - lo;
#pragma unroll
    for (int k = 0; k < MC_ITEMS; ++k) {
      const u64 x = s[ia < la ? ia : 0], y = s[la + (ib < lb ? ib : 0)];
      const bool ta = ia < la && (ib >= lb || x <= y);
      v[k] = ta ? x : y;
      ia += ta ? 1u : 0u;
      ib += ta ? 0u : 1u;
    }
  }
  __syncthreads();
#pragma unroll
  for (int k = 0; k < MC_ITEMS; ++k)
    if (q0 + k < len) s[q0 + k] = v[k];
  __syncthreads();
  for (u32 t = threadIdx.x; t < len; t += MC_THREADS) out[r0 + t] = s[t];
}

int merge_copy_device(const u64* a, u64 na, const u64* b, u64 nb, u64* out, cudaStream_t st) {
  const u64 n = na + nb;
  if (n == 0) return PIP_OK;
  const u64 blocks = (n + MC_TILE - 1) / MC_TILE;
  if (blocks > 0x7fffffffull) return PIP_ERR_UNSUPPORTED;
  merge_copy_kernel<<<(unsigned)blocks, MC_THREADS, 0, st>>>(a, na, b, nb, out);
  PIP_CHECK_LAUNCH();
  return PIP_OK;
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
    merge_small_kernel<<<1, MG_CP, smem, st>>>(a, (u32)n, (u32)split);
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
  M.rlo = (u32*)(w + L.rlo);
  M.rhi = (u32*)(w + L.rhi);
  M.cr = (u64*)(w + L.cr);
  M.plan = (ulonglong4*)(w + L.plan);
  // the per-CTA load status words live in the caller's O(#CTAs) device
  // scratch (like the scan look-back ring), not in the metered workspace
  const size_t status_off = 128, status_bytes = (size_t)grid * 4 * MG_SST;
  if (!scratch || scratch_bytes < status_off + status_bytes) return PIP_ERR_OOM;
  M.status = (u32*)((char*)scratch + status_off);
  M.head_save = (u64*)(w + L.head);
  M.g = (MergeGlobal*)(w + L.g);
  if ((u64)grid <= 2 * M.L || grid > 256) return PIP_ERR_UNSUPPORTED;
  PIP_CUDA(cudaMemsetAsync(M.status, 0, status_bytes, st));
  PIP_CUDA(cudaMemsetAsync(M.g, 0, sizeof(MergeGlobal), st));
  const size_t smem = MG_SMEM;
  PIP_CUDA(cudaFuncSetAttribute(merge_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  void* args[] = {&M};
  PIP_CUDA(cudaLaunchCooperativeKernel((const void*)merge_kernel, dim3(grid), dim3(MG_THREADS), args,
                                       smem, st));
  MergeGlobal gh{};
  PIP_CUDA(cudaMemcpyAsync(&gh, M.g, sizeof(gh), cudaMemcpyDeviceToHost, st));
  PIP_CUDA(cudaStreamSynchronize(st));
  if (gh.sync.abort) return PIP_ERR_STALLED;
  if (timing_enabled() && (M.dbg & 4))
    fprintf(stderr, "[pip merge] CTA0 cycles: merge warps: wait data %llu | merge %llu | wait output buffer %llu | write-out %llu ; "
            "loader: refills/publishes %llu | watcher: dataflow wait %llu | missing-reader polls after m %llu before m %llu\n",
            (unsigned long long)gh.sec[0], (unsigned long long)gh.sec[1], (unsigned long long)gh.sec[2],
            (unsigned long long)gh.sec[3], (unsigned long long)gh.sec[4], (unsigned long long)gh.sec[5],
            (unsigned long long)gh.sec[6], (unsigned long long)gh.sec[7]);
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
