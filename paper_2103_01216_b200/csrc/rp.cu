// In-place random permutation by deterministic reservations
// (relaxed.random_permutation on detres.run_rounds).
//
// Reference: pkg/src/pipal/relaxed.py:64-251 (_RpClient: next_ids :107-120,
// reserve :130-159, commit :161-197, clean :199-217) and
// pkg/src/pipal/detres.py:40-211 (ReservationTable), :256-307 (run_rounds).
//
// Semantics kept bit-for-bit (so rounds, committed-per-round, trace and
// peak_table_load equal the reference's):
//   * iterates are ids i with H[i] != i taken in DESCENDING order from a
//     window [cursor - W + 1, cursor] (W = span_cap = b + b/4 + 8 for
//     `final`, max(count, 1024) otherwise), at most `count = b - #failures`
//     per round; an empty window advances the cursor (next_ids);
//   * failures of a round are packed first, in order (compact_by_mask);
//   * reserve: R[H[i]] = max(R[H[i]], i) (naive/flat also R[i] = max(., i));
//     `final` serves targets inside this round's fresh id range [dlo, dhi]
//     from a dense array (slot = 1 + writer id), all others from an
//     open-addressed, linear-probed write-max table keyed by
//     (k * GOLDEN) >> (64 - log2 cap), cap = pow2 >= 2b (4b naive/flat);
//   * commit: i commits iff nobody active targets i (own slot empty or i)
//     and i holds its target's reservation; then swap a[i], a[H[i]];
//   * livelock after 64 zero-commit rounds.
//
// B200 design: ONE cooperative persistent kernel runs every round; the four
// phases of a round (pack+clean+window-count | refill | reserve | commit)
// are separated by a grid barrier, so a round costs four barriers instead
// of host round-trips.  Reservations are single 64-bit words
// (key << 32 | id): claim = atomicCAS on the empty word, update =
// atomicMax on the same word (same key => max on the id).  The slot each
// target landed in is remembered, so the commit check and the targeted
// clean are single accesses with no re-probing.  All per-iterate state is
// 32-bit (n < 2^32 - 1) to halve the workspace traffic.
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <vector>
#include <chrono>
#include <thread>
#include "sync.cuh"

namespace pip {

static constexpr int RP_THREADS = 256;
static constexpr u64 RP_EMPTY = ~0ull;
static constexpr u32 RP_NOSLOT = 0xffffffffu;
static constexpr u32 RP_TMASK = 0x7fffffffu;  // BM 1: tg bit 31 = first marker
static constexpr u64 RP_ROUND_CHUNK = 512;  // committed counts per launch

struct RpGlobal {
  GridSync sync;  // barrier + abort + kernel error (PIP_ERR_*)
  u64 dlo, dhi;
  u64 t[4];       // ns accumulated per phase by CTA 0 (P1 retire, P2 refill, P3 reserve, P4 commit)
  u64 ticket;     // scheme 3: next shared piece of the commit pass
  u64 wsum[5];    // -DPIP_RP_WAITSTAT: ns every CTA spent inside each of scheme 3's 5 barriers, summed
};

struct RpResume {
  u64 fill, rounds, zero_rounds, total_committed, peak, trace_pos, nfail_prev;
  long long cursor;
  u64 dlo, dhi;
  u32 ping, done, first, logcap_c;  // logcap_c: BM collided-table size of the last round
  u32 wpre, pad;                     // wpre: wcnt already holds the counts of the window at `cursor`
  u64 rlo, rhi;                      // BM 3: id range of the last round's active list (marked in B)
};

struct RpArgs {
  u64* a;
  const u64* h;
  u64 n, prefix, span_cap, rounds_limit;
  u32 logcap, debug, targeted_clean_ok, pad;
  u32* ids[2];
  u32* tg[2];
  u32* slot;
  unsigned char* cflag;
  u32* dense;
  u64* table;
  u32* failcnt;
  u32* wcnt;
  u32* claimcnt;
  u64* round_counts;  // RP_ROUND_CHUNK
  // host-mapped word (NULL = off): after every round, the highest id still
  // pending; a[id + 1 : n) is final (iterate i only touches a[i] and
  // a[H[i]] with H[i] <= i) and may be copied out while the rounds go on
  u64* progress;
  u64* trace;
  RpGlobal* g;
  RpResume* resume;
  u32* bmB;  // BM: bit t set <=> some active iterate targets t this round
  u32* bmC;  // BM 1: bit t set <=> at least two active iterates target t
  u32* lc;   // BM 2: per-CTA lists of iterates whose target was already marked
  u32* lccnt;  // BM: list lengths [G]
  u64 bm_words;
  // BM 3: collisions are detected on a FOLDED bitmap bmF of 2^logf bits
  // (bit t & (2^logf - 1), L2-resident); B only receives the targets inside
  // the active id range (the own checks), a narrow, L2-resident band of it
  u32* bmF;
  u32 logf, dbg;
  u32 steal_pct, pad2;  // scheme 3: share of every part handed out by ticket in the commit pass
  u32 wf, wn;  // scheme 3: weights of a carried-over failure / a fresh iterate in the list split
  u32 tload, pad5;  // collided table: slots per listed iterate (BM 2/3)
  // BM 2/3: listed-key filter, bit (t mod 2^RP_LF_LOG2) set for every listed
  // target, so a first marker probes the collided table only when its bit
  // is set (NULL = probe always)
  u32* lf;
  u32* claim2;  // BM 3: per-CTA correction of the distinct-target count
  // non-self count of every 2^RP_BLK_SHIFT-id block of H (from the validation
  // pass), so the window counts need no second read of H (NULL = read H)
  const u32* bcnt;
  // validation counts {non-self iterates, invalid targets}, written on the
  // device by the validation pass just before the launch (NULL = the host
  // read them already and set `prefix` = min(prefix, non-self))
  const u64* vcnt;
};
static constexpr u32 RP_BLK_SHIFT = 12;
#ifndef PIP_RP_LF_LOG2
#define PIP_RP_LF_LOG2 24
#endif
static constexpr u32 RP_LF_LOG2 = PIP_RP_LF_LOG2;  // 2 MiB filter

__device__ __forceinline__ void part(u64 total, u32 G, u32 b, u64& s, u64& e) {
  s = total * b / G;
  e = total * (b + 1) / G;
}

// The round's list is [failures of the previous round | fresh iterates].
// Split it among the CTAs by WEIGHT (wf per failure, wn per fresh iterate):
// a fresh iterate commits -- and pays for a DRAM exchange -- more often than
// one that has already failed, so an even split leaves the CTAs of the
// failure part idle at the end of the commit pass.  Every phase of a round
// (marks, commit, resolve and the next round's retire) uses the same split.
__device__ __forceinline__ void lpart(u64 total, u64 nf, u32 wf, u32 wn, u32 G, u32 b, u64& s, u64& e) {
  if (wf == wn) {
    part(total, G, b, s, e);
    return;
  }
  if (nf > total) nf = total;
  const u64 Wf = nf * wf, W = Wf + (total - nf) * wn;
  auto at = [&](u64 w) -> u64 { return w <= Wf ? w / wf : nf + (w - Wf) / wn; };
  s = at(W * b / G);
  e = b + 1 == G ? total : at(W * (b + 1) / G);
}

// block-wide stable exclusive rank of `f`; *tot = number of set flags
__device__ __forceinline__ u32 block_rank(bool f, u32* s_cnt, u32* tot) {
  const u32 lane = lane_id(), warp = warp_id();
  const u32 m = __ballot_sync(0xffffffffu, f);
  const u32 wr = __popc(m & ((1u << lane) - 1u));
  if (lane == 0) s_cnt[warp] = __popc(m);
  __syncthreads();
  if (warp == 0) {
    const u32 nw = blockDim.x / 32;
    u32 v = lane < nw ? s_cnt[lane] : 0;
    u32 inc = v;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      u32 t = __shfl_up_sync(0xffffffffu, inc, o);
      if (lane >= (u32)o) inc += t;
    }
    if (lane < nw) s_cnt[lane] = inc - v;
    if (lane == 31) s_cnt[32] = inc;
  }
  __syncthreads();
  const u32 r = s_cnt[warp] + wr;
  *tot = s_cnt[32];
  __syncthreads();
  return r;
}

// signed sum of the int32 words cnt[0..G) (all threads get it)
__device__ __forceinline__ long long sum_counts_signed(const u32* cnt, u32 G, u64* s_red) {
  if (threadIdx.x < 32) {
    long long t = 0;
    for (u32 i = threadIdx.x; i < G; i += 32) t += (int)__ldcg(cnt + i);
#pragma unroll
    for (int o = 16; o; o >>= 1) t += __shfl_down_sync(0xffffffffu, t, o);
    if (threadIdx.x == 0) s_red[35] = (u64)t;
  }
  __syncthreads();
  const long long r = (long long)s_red[35];
  __syncthreads();
  return r;
}

// block-wide exclusive prefix of per-thread counts v (< 2^16 each); *tot = sum
__device__ __forceinline__ u32 block_excl_sum(u32 v, u32* s_cnt, u32* tot) {
  const u32 lane = lane_id(), warp = warp_id();
  u32 inc = v;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const u32 t = __shfl_up_sync(0xffffffffu, inc, o);
    if (lane >= (u32)o) inc += t;
  }
  if (lane == 31) s_cnt[warp] = inc;
  __syncthreads();
  if (warp == 0) {
    const u32 nw = blockDim.x / 32;
    const u32 w = lane < nw ? s_cnt[lane] : 0;
    u32 wi = w;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const u32 t = __shfl_up_sync(0xffffffffu, wi, o);
      if (lane >= (u32)o) wi += t;
    }
    if (lane < nw) s_cnt[lane] = wi - w;
    if (lane == 31) s_cnt[32] = wi;
  }
  __syncthreads();
  const u32 r = s_cnt[warp] + inc - v;
  *tot = s_cnt[32];
  __syncthreads();
  return r;
}

// items per thread per pass in the latency-bound loops (independent loads in flight)
static constexpr int RB_DEFAULT = 4;
#ifndef PIP_RP_RB3
#define PIP_RP_RB3 2  // the same for scheme 3: at 8 CTAs per SM (32 registers) 2 spill least (C4 116.7 ms; 4: 120.5, 1: 120.7)
#endif

__device__ __forceinline__ u64 block_sum(u64 v, u64* s_red) {
  v = warp_reduce<Op<PIP_OP_ADD>>(v);
  if (lane_id() == 0) s_red[warp_id()] = v;
  __syncthreads();
  u64 t = 0;
  if (threadIdx.x == 0) {
    for (u32 w = 0; w < blockDim.x / 32; ++w) t += s_red[w];
    s_red[32] = t;
  }
  __syncthreads();
  t = s_red[32];
  __syncthreads();
  return t;
}

// sum of cnt[0..G) and exclusive prefix up to b (all threads get both)
__device__ __forceinline__ void sum_counts(const u32* cnt, u32 G, u32 b, u64* s_red, u64& total,
                                           u64& before) {
  if (threadIdx.x < 32) {
    u64 t = 0, bf = 0;
    for (u32 i = threadIdx.x; i < G; i += 32) {
      const u64 v = __ldcg(cnt + i);
      t += v;
      if (i < b) bf += v;
    }
    t = warp_reduce<Op<PIP_OP_ADD>>(t);
    bf = warp_reduce<Op<PIP_OP_ADD>>(bf);
    if (threadIdx.x == 0) {
      s_red[33] = t;
      s_red[34] = bf;
    }
  }
  __syncthreads();
  total = s_red[33];
  before = s_red[34];
  __syncthreads();
}

// sum of cnt[0..G), exclusive prefix up to b, and the sum of cnt2[0..G)
__device__ __forceinline__ void sum_counts2(const u32* cnt, const u32* cnt2, u32 G, u32 b, u64* s_red,
                                            u64& total, u64& before, u64& total2) {
  if (threadIdx.x < 32) {
    u64 t = 0, bf = 0, t2 = 0;
    for (u32 i = threadIdx.x; i < G; i += 32) {
      const u64 v = __ldcg(cnt + i);
      t2 += __ldcg(cnt2 + i);
      t += v;
      if (i < b) bf += v;
    }
    t = warp_reduce<Op<PIP_OP_ADD>>(t);
    bf = warp_reduce<Op<PIP_OP_ADD>>(bf);
    t2 = warp_reduce<Op<PIP_OP_ADD>>(t2);
    if (threadIdx.x == 0) {
      s_red[33] = t;
      s_red[34] = bf;
      s_red[35] = t2;
    }
  }
  __syncthreads();
  total = s_red[33];
  before = s_red[34];
  total2 = s_red[35];
  __syncthreads();
}

// non-self ids in [x, y] (inclusive), summed over the CTA: whole blocks from
// the block counts, the ragged ends from H itself
__device__ __forceinline__ u64 count_nonself_range(const RpArgs& A, u64 x, u64 y) {
  if (x > y) return 0;
  u64 c = 0;
  const u64 B = 1ull << RP_BLK_SHIFT;
  const u64 fb = (x + B - 1) >> RP_BLK_SHIFT, lb = (y + 1) >> RP_BLK_SHIFT;  // full blocks [fb, lb)
  if (A.bcnt && fb < lb) {
    for (u64 q = fb + threadIdx.x; q < lb; q += blockDim.x) c += __ldg(A.bcnt + q);
    const u64 e1 = fb << RP_BLK_SHIFT, s2 = lb << RP_BLK_SHIFT;
    for (u64 id = x + threadIdx.x; id < e1; id += blockDim.x) c += __ldcs(A.h + id) != id;
    for (u64 id = s2 + threadIdx.x; id <= y; id += blockDim.x) c += __ldcs(A.h + id) != id;
  } else {
    for (u64 id = x + threadIdx.x; id <= y; id += blockDim.x) c += __ldcs(A.h + id) != id;
  }
  return c;
}

// ---------------------------------------------------------------------------
// The swap of a committed iterate.  A round's committed swaps touch disjoint
// words (each word is reserved by exactly one committing iterate), so the
// random side may be ONE atomic exchange (one request through the SM's
// load/store queue and one L2 read-modify-write) instead of a load and a
// store: 20.1 against 14.9 G random updates/s over 8 GiB (tools/rmw_modes.py).
// Scheme 3 (n > 2^28, DRAM-bound swaps) exchanges; the small-n schemes keep
// the load + store form, whose two loads travel together (C0: 1.51 against
// 1.56 ms).  PIP_RP_DBG bit 1 flips the choice (measurement knob).
template <int BM>
__device__ __forceinline__ void rp_swap(u64* a, u32 i, u32 t, u32 dbg) {
  if ((BM == 3) != ((dbg & 2u) != 0)) {
    const u64 x = __ldcg(a + i);
    a[i] = (u64)atomicExch((unsigned long long*)a + t, (unsigned long long)x);
  } else {
    const u64 x = __ldcg(a + i), y = __ldcg(a + t);
    a[i] = y;
    a[t] = x;
  }
}

// ---------------------------------------------------------------------------
// write-max reservation table: one 64-bit word per slot, key<<32 | value
__device__ __forceinline__ u64 rp_home(u32 key, u32 logcap) {
  return ((u64)key * GOLDEN) >> (64 - logcap);
}

__device__ __forceinline__ u32 table_reserve(u64* table, u32 logcap, u32 key, u32 val,
                                             u32& claimed, u32* err) {
  const u64 mask = (1ull << logcap) - 1;
  u64 s = rp_home(key, logcap);
  const u64 want = ((u64)key << 32) | val;
  for (u64 step = 0; step <= mask; ++step) {
    u64 cur = __ldcg(table + s);
    if (cur == RP_EMPTY) {
      const u64 prev = atomicCAS(reinterpret_cast<unsigned long long*>(table + s), RP_EMPTY, want);
      if (prev == RP_EMPTY) {
        claimed += 1;
        return (u32)s;
      }
      cur = prev;
    }
    if ((u32)(cur >> 32) == key) {
      if ((u32)cur < val) atomicMax(reinterpret_cast<unsigned long long*>(table + s), want);
      return (u32)s;
    }
    s = (s + 1) & mask;
  }
  atomicExch(err, (u32)PIP_ERR_TABLE);
  return RP_NOSLOT;
}

__device__ __forceinline__ bool table_lookup(const u64* table, u32 logcap, u32 key, u32& val) {
  const u64 mask = (1ull << logcap) - 1;
  u64 s = rp_home(key, logcap);
  for (u64 step = 0; step <= mask; ++step) {
    const u64 cur = __ldcg(table + s);
    if (cur == RP_EMPTY) return false;
    if ((u32)(cur >> 32) == key) {
      val = (u32)cur;
      return true;
    }
    s = (s + 1) & mask;
  }
  return false;
}

// ---------------------------------------------------------------------------
// BM (final variant, budget permitting): reservations by a bitmap.  Almost
// every target of a round is hit by exactly one iterate.  B[t] records "t is
// targeted" (own check: i may commit only if !B[i]); an iterate whose
// atomicOr finds B[t] already set goes to a per-CTA list, and only those
// iterates (plus the first marker of their targets) use the write-max table,
// sized per round for them alone so that it stays L2-resident.  Same commit
// rule, so the same rounds as the reference.
#ifndef PIP_RP_WF_DEFAULT
#define PIP_RP_WF_DEFAULT 5  // measured at C4: 5:4 116.05 ms, 4:4 116.7, 6:4 116.7, 4:5 121.0
#define PIP_RP_WN_DEFAULT 4
#endif
#ifndef PIP_RP_STEAL_DEFAULT
#define PIP_RP_STEAL_DEFAULT 30
#endif
#ifndef PIP_RP_STEAL_STEPS
#define PIP_RP_STEAL_STEPS 4  // steps of 256 items per shared piece (C4: 1: 115.7 ms, 2: 113.3, 4: 112.5, 8: 113.2)
#endif
static constexpr int RP_STEAL_STEPS = PIP_RP_STEAL_STEPS;
#ifndef PIP_RP_WAITSTAT
#define PIP_RP_WAITSTAT 0  // measurement build: time every CTA spends inside the barriers
#endif
#ifndef PIP_RP_SPEC1
#define PIP_RP_SPEC1 1
#endif
#ifndef PIP_RP_SMALL1
#define PIP_RP_SMALL1 1
#endif
#ifndef PIP_RP_PF3
#define PIP_RP_PF3 0  // scheme 3: retire / refill loops load their next batch early (at 6 CTAs per SM it no longer pays: 118.9 vs 118.5 ms)
#endif
#ifndef PIP_RP_XPRE
#define PIP_RP_XPRE 1
#endif
#ifndef PIP_RP_MINB3
#define PIP_RP_MINB3 8  // resident CTAs per SM of the scheme-3 kernel (32 registers; 6: 40, 4: 64)
#endif
// MB: resident CTAs per SM the kernel is compiled for.  MB = 1 (scheme 1
// only) is the flavour for grids of at most one CTA per SM (C0: 79 CTAs):
// no register cap, so nothing spills into the rounds' latency chains.
template <int V, int BM, int MB = (BM == 3 ? PIP_RP_MINB3 : 4)>
__global__ void __launch_bounds__(RP_THREADS, MB) rp_kernel(RpArgs A) {
  __shared__ u32 s_cnt[33];
  __shared__ u64 s_red[36];
  constexpr int RB = BM == 3 ? PIP_RP_RB3 : RB_DEFAULT;
  const u32 b = blockIdx.x, G = gridDim.x, tid = threadIdx.x, T = blockDim.x;
  RpGlobal* g = A.g;
  // The round state (identical in every thread) is touched only between
  // phases.  Scheme 3 keeps it in shared memory, written by thread 0 between
  // two CTA barriers (RSET), so the phase loops have ~30 more registers and
  // the kernel fits 6 CTAs per SM; the small-n schemes keep it in registers
  // (their rounds are latency-bound: the extra barriers would show).
  __shared__ RpResume s_R;
  RpResume R_reg;
  RpResume& R = (BM == 3) ? s_R : R_reg;
  if (BM == 3) {
    if (tid == 0) s_R = *A.resume;
    __syncthreads();
  } else {
    R_reg = *A.resume;
  }
#define RSET(...)                              \
  do {                                         \
    if (BM == 3) __syncthreads();              \
    if (BM != 3 || tid == 0) { __VA_ARGS__; }  \
    if (BM == 3) __syncthreads();              \
  } while (0)
  u64 P = A.prefix;  // run_rounds clamps the active prefix to n_iterates (detres.py:267)
  if (A.vcnt) {
    const u64 ns = __ldcg(A.vcnt), bad = __ldcg(A.vcnt + 1);
    if (bad || ns == 0) {  // nothing to do, or invalid H: a[] is not touched
      if (b == 0 && tid == 0) {
        R.done = 1;
        *A.resume = R;
      }
      return;
    }
    if (ns < P) P = ns;
  }
  u32 gen = 0;
#if PIP_RP_WAITSTAT
  u64 wacc[5] = {0, 0, 0, 0, 0}, wt0 = 0;
#define WSTAT_T0() do { if (tid == 0) wt0 = globaltimer_ns(); } while (0)
#define WSTAT_T1(i) do { if (tid == 0) wacc[i] += globaltimer_ns() - wt0; } while (0)
#else
#define WSTAT_T0() do { } while (0)
#define WSTAT_T1(i) do { } while (0)
#endif
  u64 rounds_here = 0;
  const bool trace = A.trace != nullptr;
  const bool tm = b == 0 && tid == 0;
  // phase timers of CTA 0 (PIP_TIMING): shared memory, so they take no registers
  __shared__ u64 s_tacc[5];
  if (tm) {
    s_tacc[0] = s_tacc[1] = s_tacc[2] = s_tacc[3] = 0;
    s_tacc[4] = globaltimer_ns();
  }
  auto tick = [&](int ph) {
    if (tm) {
      const u64 now = globaltimer_ns();
      s_tacc[ph] += now - s_tacc[4];
      s_tacc[4] = now;
    }
  };

  while (!R.done) {
    // ======================= P1: retire previous round =====================
    const u32 old = R.ping, nw = R.ping ^ 1u;
    // BM 1: two bitmap pairs by round parity.  This round marks and reads
    // (Bc, Cc); its failures mark the NEXT round's targets in (Bp, Cp) as
    // soon as they fail, and the fresh ids mark during the refill, so no
    // separate mark phase (and no grid barrier for it) is needed.  (Bp, Cp)
    // held the previous round's marks and are cleared by the retire below.
    const u64 pofs = BM == 1 ? (R.rounds & 1u) * A.bm_words : 0, qofs = BM == 1 ? A.bm_words - pofs : 0;
    u32* const Bc = A.bmB + pofs;
    u32* const Cc = A.bmC + pofs;
    u32* const Bp = A.bmB + qofs;
    u32* const Cp = A.bmC + qofs;
    const u32* ids_o = A.ids[old];
    const u32* tg_o = A.tg[old];
    u32* ids_n = A.ids[nw];
    u32* tg_n = A.tg[nw];
    u64 nfail = 0;
    if (!R.first) {
      const u64 F = R.fill;
      u64 fbefore;
      if (BM == 1) {
        // the previous round's distinct out-of-window targets ride along
        u64 claims_total;
        sum_counts2(A.failcnt, A.claimcnt, G, b, s_red, nfail, fbefore, claims_total);
        RSET(if (claims_total > R.peak) R.peak = claims_total);
      } else {
        sum_counts(A.failcnt, G, b, s_red, nfail, fbefore);
      }
      const u64 ncommit = F - nfail;
      // committed-per-round + livelock bookkeeping (identical in every CTA)
      if (b == 0 && tid == 0) {
        const u64 r = R.rounds - 1;
        A.round_counts[r % RP_ROUND_CHUNK] = ncommit;
      }
      RSET(R.total_committed += ncommit; R.zero_rounds = ncommit == 0 ? R.zero_rounds + 1 : 0);
      if (R.zero_rounds >= 64) {
        if (b == 0 && tid == 0) atomicExch(&g->sync.error, (u32)PIP_ERR_LIVELOCK);
        RSET(R.done = 1);
        break;
      }
      u64 s, e;
      if (BM == 3) lpart(F, R.nfail_prev, A.wf, A.wn, G, b, s, e);
      else part(F, G, b, s, e);
      const u64 cbefore = s - fbefore;  // committed items in CTAs < b
      const bool targeted = A.targeted_clean_ok && F * 8 < (1ull << A.logcap);
      u64 runf = 0, runc = 0;
      const u64 trace_pos0 = R.trace_pos;
      // RB consecutive items per thread: failures keep their order; the
      // next batch's loads are in flight while this batch is packed
      u32 cn[RB], inx[RB], tnx[RB];
#pragma unroll
      for (int q = 0; q < RB; ++q) {
        const u64 k = s + (u64)RB * tid + q;
        cn[q] = 1;
        inx[q] = tnx[q] = 0;
        if (k < e) {
          cn[q] = __ldcs(A.cflag + k);
          inx[q] = __ldcs(ids_o + k);
          tnx[q] = __ldcs(tg_o + k);
        }
      }
      for (u64 c0 = s; c0 < e; c0 += (u64)RB * T) {
        const u64 kb = c0 + (u64)RB * tid;
        u32 fm = 0, cm = 0, iv[RB], tv[RB];
        if (!(BM == 3 && PIP_RP_PF3) && c0 != s) {
#pragma unroll
          for (int q = 0; q < RB; ++q) {
            const u64 k = kb + q;
            if (k < e) {
              cn[q] = __ldcs(A.cflag + k);
              inx[q] = __ldcs(ids_o + k);
              tnx[q] = __ldcs(tg_o + k);
            }
          }
        }
#pragma unroll
        for (int q = 0; q < RB; ++q) {
          iv[q] = inx[q];
          tv[q] = tnx[q];
          if (kb + q < e) {
            if (BM == 1 ? (cn[q] & 1u) : cn[q]) cm |= 1u << q;
            else fm |= 1u << q;
          }
          // BM 1: bit 2 = the failure was its next-round target's first marker
          // (tg bit 31 in the new list); bit 3 = it holds a table slot
          if (BM == 1) tv[q] = (tv[q] & RP_TMASK) | ((u32)(cn[q] & 4u) << 29);
        }
        u32 cf1[RB];
#pragma unroll
        for (int q = 0; q < RB; ++q) cf1[q] = cn[q];
        // (scheme 3 only: the large rounds of C4 gain 0.8 ms; at C0's size the
        // extra live registers spill and cost more than they hide)
        if (BM == 3 && PIP_RP_PF3) {
#pragma unroll
          for (int q = 0; q < RB; ++q) {
            const u64 k = kb + (u64)RB * T + q;
            if (k < e) {
              cn[q] = __ldcs(A.cflag + k);
              inx[q] = __ldcs(ids_o + k);
              tnx[q] = __ldcs(tg_o + k);
            }
          }
        }
        u32 tot;
        u64 pos = fbefore + runf + block_excl_sum(__popc(fm), s_cnt, &tot);
#pragma unroll
        for (int q = 0; q < RB; ++q)
          if ((fm >> q) & 1u) {
            ids_n[pos] = iv[q];
            tg_n[pos] = tv[q];
            ++pos;
          }
        runf += tot;
        if (trace) {
          u32 totc;
          u64 cp = trace_pos0 + cbefore + runc + block_excl_sum(__popc(cm), s_cnt, &totc);
#pragma unroll
          for (int q = 0; q < RB; ++q)
            if ((cm >> q) & 1u) A.trace[cp++] = iv[q];
          runc += totc;
        }
#pragma unroll
        for (int q = 0; q < RB; ++q) {
          const u64 k = kb + q;
          if (k >= e) continue;
          if (BM == 1) {
            if (cf1[q] & 8u) A.table[__ldcg(A.slot + k)] = RP_EMPTY;
          } else if (!BM && targeted) {
            const u32 sl = __ldcg(A.slot + k);
            if (sl != RP_NOSLOT) A.table[sl] = RP_EMPTY;
          }
          if (BM && BM != 3 && F * 256 < A.n) {  // sparse round: clear the touched words
            const u32 tq = tv[q] & RP_TMASK;
            Bp[tq >> 5] = 0u;
            if (BM == 1) Cp[tq >> 5] = 0u;
          }
        }
      }
      RSET(R.trace_pos += ncommit);
      if (BM == 3) {
        // the folded bitmap wholesale (L2-resident); B only over the band of
        // ids the last round marked
        u64 ts, te;
        part(1ull << (A.logf - 5), G, b, ts, te);
        for (u64 x = ts + tid; x < te; x += T) A.bmF[x] = 0u;
        const u64 rlo = R.rlo, rhi = R.rhi;
        if (rhi >= rlo) {
          part((rhi >> 5) - (rlo >> 5) + 1, G, b, ts, te);
          for (u64 x = ts + tid; x < te; x += T) A.bmB[(rlo >> 5) + x] = 0u;
        }
      }
      if (BM && BM != 3 && F * 256 >= A.n) {  // dense round: clear the bitmaps wholesale
        u64 ts, te;
        part(A.bm_words, G, b, ts, te);
        for (u64 x = ts + tid; x < te; x += T) {
          Bp[x] = 0u;
          if (BM == 1) Cp[x] = 0u;
        }
      }
      if ((BM == 2 || BM == 3) && R.logcap_c && A.lf) {
        u64 ts, te;
        part(1ull << (RP_LF_LOG2 - 5), G, b, ts, te);
        for (u64 x = ts + tid; x < te; x += T) A.lf[x] = 0u;
      }
      if ((BM == 2 || BM == 3) && R.logcap_c) {  // the collided table used only its first 2^logcap_c slots
        u64 ts, te;
        part(1ull << (u32)R.logcap_c, G, b, ts, te);
        for (u64 x = ts + tid; x < te; x += T) A.table[x] = RP_EMPTY;
      }
      if (!targeted && !BM) {
        const u64 cap = 1ull << A.logcap;
        u64 ts, te;
        part(cap, G, b, ts, te);
        for (u64 x = ts + tid; x < te; x += T) A.table[x] = RP_EMPTY;
      }
      if (V == PIP_RP_FINAL && !BM && R.dhi >= R.dlo) {
        u64 ds, de;
        const u64 odlo = R.dlo, odhi = R.dhi;
        part(odhi - odlo + 1, G, b, ds, de);
        for (u64 x = ds + tid; x < de; x += T) A.dense[x] = 0;
      }
    }
    // window for the refill (next_ids)
    const u64 count = P - nfail;
    long long cursor = R.cursor;
    u64 hi = 0, lo = 0, wd = 0;
    bool win = count > 0 && cursor >= 0;
    auto count_window = [&]() {
      hi = (u64)cursor;
      const u64 W = (V == PIP_RP_FINAL) ? A.span_cap : (count > 1024 ? count : 1024);
      lo = hi + 1 >= W ? hi + 1 - W : 0;
      wd = hi - lo + 1;
      u64 s, e;
      part(wd, G, b, s, e);
      u64 c = e > s ? count_nonself_range(A, hi - (e - 1), hi - s) : 0;
      c = block_sum(c, s_red);
      if (tid == 0) A.wcnt[b] = (u32)c;
    };
    // `final` windows do not depend on the failures, so the previous round
    // counted this one already and retire + refill share one phase (the
    // refill writes past nfail, the retire below it; nfail comes from the
    // previous round's counts)
    const bool fused = V == PIP_RP_FINAL && R.wpre && !A.debug;
    if (fused) {
      if (win) {
        hi = (u64)cursor;
        lo = hi + 1 >= A.span_cap ? hi + 1 - A.span_cap : 0;
        wd = hi - lo + 1;
      }
    } else {
      if (win) count_window();
      if (!grid_barrier(&g->sync, gen)) break;
    }
    tick(0);

    // ======================= P2: refill =====================================
    if (A.debug && !R.first) {
      // relaxed.py:212-217: every slot touched must read as empty again
      const u64 cap = 1ull << A.logcap;
      u64 ts, te;
      part(cap, G, b, ts, te);
      for (u64 x = ts + tid; x < te; x += T)
        if (__ldcg(A.table + x) != RP_EMPTY) atomicExch(&g->sync.error, (u32)PIP_ERR_DEBUG_SWEEP);
      if (V == PIP_RP_FINAL && !BM) {
        part(A.span_cap, G, b, ts, te);
        for (u64 x = ts + tid; x < te; x += T)
          if (__ldcg(A.dense + x) != 0) atomicExch(&g->sync.error, (u32)PIP_ERR_DEBUG_SWEEP);
      }
      if (BM) {
        part(A.bm_words, G, b, ts, te);
        for (u64 x = ts + tid; x < te; x += T)
          if (__ldcg(Bp + x) | (BM == 1 ? __ldcg(Cp + x) : 0u)) atomicExch(&g->sync.error, (u32)PIP_ERR_DEBUG_SWEEP);
        if (BM == 3) {
          part(1ull << (A.logf - 5), G, b, ts, te);
          for (u64 x = ts + tid; x < te; x += T)
            if (__ldcg(A.bmF + x)) atomicExch(&g->sync.error, (u32)PIP_ERR_DEBUG_SWEEP);
        }
      }
    }
    u64 total_ns = 0, wbefore = 0;
    bool aborted = false;
    while (win) {
      sum_counts(A.wcnt, G, b, s_red, total_ns, wbefore);
      if (total_ns > 0) break;
      cursor = (long long)lo - 1;  // empty window: move on (relaxed.py:119)
      win = cursor >= 0;
      if (win) count_window();
      if (!grid_barrier(&g->sync, gen)) { aborted = true; break; }
    }
    if (aborted) break;
    const u64 fresh = win ? (count < total_ns ? count : total_ns) : 0;
    if (fresh > 0) {
      u64 s, e;
      part(wd, G, b, s, e);
      u64 run = wbefore;
      if (BM == 3 && A.bcnt && !(A.dbg & 4u)) {
        // The window holds span_cap ids but only its first `fresh` non-self
        // ids are taken (about a third of it), so with the window split
        // evenly two thirds of the CTAs would have nothing to rank.  Split
        // the NEEDED stretch instead: the old parts 0..bl hold the first
        // `fresh` non-self ids (their counts are in wcnt); its whole
        // 4096-id blocks are dealt evenly to all CTAs, and a CTA's first
        // rank is the non-self count of the ids above its blocks (block
        // counts of the validation pass + the window's ragged top from H).
        const u32 per = (G + T - 1) / T;
        const u32 q0 = tid * per, q1 = q0 + per < G ? q0 + per : G;
        u32 mysum = 0;
        for (u32 q = q0; q < q1; ++q) mysum += __ldcg(A.wcnt + q);
        u32 tot0;
        const u64 pre = block_excl_sum(mysum, s_cnt, &tot0);
        if (tid == 0) s_red[32] = G - 1;
        __syncthreads();
        if (pre < fresh && pre + mysum >= fresh) {
          u64 c = pre;
          for (u32 q = q0; q < q1; ++q) {
            c += __ldcg(A.wcnt + q);
            if (c >= fresh) {
              s_red[32] = q;
              break;
            }
          }
        }
        __syncthreads();
        const u32 bl = (u32)s_red[32];
        __syncthreads();
        u64 ps, pe;
        part(wd, G, bl, ps, pe);  // positions [0, pe) cover the needed ids
        const u64 low_id = hi - (pe - 1);
        const u64 bhi = hi >> RP_BLK_SHIFT, blo = low_id >> RP_BLK_SHIFT;
        u64 bs, be;
        part(bhi - blo + 1, G, b, bs, be);  // my blocks, counted from the top
        if (be > bs) {
          u64 top = ((bhi - bs) << RP_BLK_SHIFT) + ((1ull << RP_BLK_SHIFT) - 1);
          if (top > hi) top = hi;
          u64 bot = (bhi - (be - 1)) << RP_BLK_SHIFT;
          if (bot < low_id) bot = low_id;
          s = hi - top;
          e = hi - bot + 1;
          run = block_sum(count_nonself_range(A, top + 1, hi), s_red);
        } else {
          s = e = 0;
          run = fresh;
        }
      }
      // the next batch's H words are in flight while this batch is ranked
      u64 hn[RB];
#pragma unroll
      for (int q = 0; q < RB; ++q) {
        const u64 qq = s + (u64)RB * tid + q;
        hn[q] = qq < e ? __ldcs(A.h + (hi - qq)) : 0;
      }
      for (u64 c0 = s; c0 < e && run < fresh; c0 += (u64)RB * T) {
        const u64 qb = c0 + (u64)RB * tid;
        u64 hv[RB];
        u32 fm = 0;
        if (!(BM == 3 && PIP_RP_PF3) && c0 != s) {  // (prefetch for scheme 3 only, as in the retire loop)
#pragma unroll
          for (int q = 0; q < RB; ++q) hn[q] = qb + q < e ? __ldcs(A.h + (hi - (qb + q))) : 0;
        }
#pragma unroll
        for (int q = 0; q < RB; ++q) {
          hv[q] = hn[q];
          if (qb + q < e && hv[q] != hi - (qb + q)) fm |= 1u << q;
        }
        if (BM == 3 && PIP_RP_PF3) {
          const u64 qn = qb + (u64)RB * T;
#pragma unroll
          for (int q = 0; q < RB; ++q) hn[q] = qn + q < e ? __ldcs(A.h + (hi - (qn + q))) : 0;
        }
        u32 tot;
        u64 rank = run + block_excl_sum(__popc(fm), s_cnt, &tot);
        u32 mk[RB];  // BM 1: the fresh iterates mark their targets here
        if (BM == 1) {
          u64 rk = rank;
#pragma unroll
          for (int q = 0; q < RB; ++q) {
            mk[q] = 0u;
            if ((fm >> q) & 1u) {
              if (rk < fresh) mk[q] = 1u;
              ++rk;
            }
          }
#pragma unroll
          for (int q = 0; q < RB; ++q)
            if (mk[q]) mk[q] = atomicOr(Bc + ((u32)hv[q] >> 5), 1u << (hv[q] & 31));
        }
#pragma unroll
        for (int q = 0; q < RB; ++q)
          if ((fm >> q) & 1u) {
            if (rank < fresh) {
              const u64 id = hi - (qb + q);
              ids_n[nfail + rank] = (u32)id;
              u32 tw = (u32)hv[q];
              if (BM == 1) {
                const u32 bit = 1u << (tw & 31);
                if (mk[q] & bit) atomicOr(Cc + (tw >> 5), bit);
                else tw |= 0x80000000u;  // first marker
              }
              tg_n[nfail + rank] = tw;
              if (rank == 0) g->dhi = id;
              if (rank == fresh - 1) g->dlo = id;
            }
            ++rank;
          }
        run += tot;
      }
    } else if (b == 0 && tid == 0) {
      g->dlo = 1;
      g->dhi = 0;
    }
    const u64 newF = nfail + fresh;
    if (newF == 0) {
      RSET(R.done = 1; R.cursor = cursor);
      break;
    }
    WSTAT_T0();
    if (!grid_barrier(&g->sync, gen)) break;
    WSTAT_T1(0);
    tick(1);

    // ======================= P3: reserve ====================================
    const u64 dlo = ld_relaxed_u64(reinterpret_cast<const u64*>(&g->dlo));
    const u64 dhi = ld_relaxed_u64(reinterpret_cast<const u64*>(&g->dhi));
    if (fresh > 0) cursor = (long long)dlo - 1;
    // BM 3: the active list is descending, so its ids span [band_lo, band_hi];
    // only targets inside that band can be some active iterate's own slot
    u64 band_lo = 1, band_hi = 0;
    if (BM == 3) {
      band_hi = __ldcg(ids_n);
      band_lo = __ldcg(ids_n + newF - 1);
    }
    {
      u64 s, e;
      if (BM == 3) lpart(newF, nfail, A.wf, A.wn, G, b, s, e);
      else part(newF, G, b, s, e);
      u32 claims = 0;
      if (BM == 1) {
        // marks already made (refill / previous round's failures)
      } else if (BM == 2) {
        // mark: first toucher of t sets B[t]; later ones go to the list.  The
        // reference's table holds the distinct out-of-window targets: count
        // first touches outside [dlo, dhi] (peak_table_load).
        if (tid == 0) s_cnt[32] = 0;
        __syncthreads();
        for (u64 k0 = s + tid; k0 < e; k0 += (u64)RB * T) {
          u32 t[RB], old[RB];
#pragma unroll
          for (int q = 0; q < RB; ++q) t[q] = k0 + q * T < e ? __ldcs(tg_n + k0 + q * T) : 0u;
#pragma unroll
          for (int q = 0; q < RB; ++q)
            old[q] = k0 + q * T < e ? atomicOr(A.bmB + (t[q] >> 5), 1u << (t[q] & 31)) : 0u;
#pragma unroll
          for (int q = 0; q < RB; ++q) {
            const u64 k = k0 + q * T;
            if (k >= e) continue;
            const bool coll = (old[q] >> (t[q] & 31)) & 1u;
            if (coll) A.lc[s + atomicAdd(s_cnt + 32, 1u)] = (u32)(k - s);
            else if (t[q] < dlo || t[q] > dhi) claims += 1;
            A.cflag[k] = coll ? 2 : 0;
          }
        }
        __syncthreads();
        if (tid == 0) A.lccnt[b] = s_cnt[32];
      } else if (BM == 3) {
        // mark: the first toucher of FOLDED bit (t mod 2^logf) is its
        // "first marker"; later touchers go to the list (every reserver of
        // a target other than its first marker lands there, plus a few that
        // only share the folded bit).  Targets inside the active band also
        // set B[t] for the own checks.
        if (tid == 0) {
          s_cnt[32] = 0;
          A.failcnt[b] = 0u;           // this round's failures are ADDED (work stealing in the commit pass)
          if (b == 0) g->ticket = 0;  // nobody draws a ticket before the barriers below
        }
        __syncthreads();
        const u32 fmask = (u32)((1ull << A.logf) - 1ull);
        u32 tn[RB];  // the next batch's targets travel while this batch marks
#pragma unroll
        for (int q = 0; q < RB; ++q) tn[q] = s + tid + q * T < e ? __ldcs(tg_n + s + tid + q * T) : 0u;
        for (u64 k0 = s + tid; k0 < e; k0 += (u64)RB * T) {
          u32 t[RB], old[RB];
#pragma unroll
          for (int q = 0; q < RB; ++q) {
            t[q] = tn[q];
            const u64 kn = k0 + (u64)RB * T + q * T;
            tn[q] = kn < e ? __ldcs(tg_n + kn) : 0u;
          }
#pragma unroll
          for (int q = 0; q < RB; ++q)
            old[q] = k0 + q * T < e ? atomicOr(A.bmF + ((t[q] & fmask) >> 5), 1u << (t[q] & 31)) : 0u;
#pragma unroll
          for (int q = 0; q < RB; ++q) {
            const u64 k = k0 + q * T;
            if (k >= e) continue;
            if (t[q] >= band_lo && t[q] <= band_hi) atomicOr(A.bmB + (t[q] >> 5), 1u << (t[q] & 31));
            const bool coll = (old[q] >> (t[q] & 31)) & 1u;
            if (coll) A.lc[s + atomicAdd(s_cnt + 32, 1u)] = (u32)(k - s);
            else if (t[q] < dlo || t[q] > dhi) claims += 1;
            A.cflag[k] = coll ? 2 : 0;
          }
        }
        __syncthreads();
        if (tid == 0) A.lccnt[b] = s_cnt[32];
      } else {
      for (u64 k = s + tid; k < e; k += T) {
        const u32 i = __ldcs(ids_n + k), t = __ldcs(tg_n + k);
        u32 sl = RP_NOSLOT;
        if (V == PIP_RP_FINAL && t >= dlo && t <= dhi) {
          atomicMax(A.dense + (dhi - t), i + 1u);
        } else {
          if (V == PIP_RP_NAIVE || V == PIP_RP_FLAT)
            table_reserve(A.table, A.logcap, i, i, claims, &g->sync.error);
          sl = table_reserve(A.table, A.logcap, t, i, claims, &g->sync.error);
        }
        A.slot[k] = sl;
      }
      }
      if (BM != 1) {
        const u64 c = block_sum(claims, s_red);
        if (tid == 0) A.claimcnt[b] = (u32)c;
      }
    }
    if (BM == 1) {
      // P3b: iterates on targets hit once (no C bit) are their target's only
      // reserver and commit now; the few on C targets reserve in the
      // write-max table and are resolved in P4 (cflag 2).  A failure marks
      // its target for the next round in (Bp, Cp) right away (cflag bit 2 =
      // first marker there).  The distinct out-of-window targets
      // (peak_table_load) are the first markers outside [dlo, dhi].
      tick(2);
      u64 s, e;
      part(newF, G, b, s, e);
      u32 fails = 0, dclaim = 0, claims1 = 0;
      // the next round's window [cursor - span + 1, cursor] is known now: its
      // H words are loaded here, in flight with this phase's chain (<= 4 per
      // thread; wider CTA shares count at the end of the round as before)
      constexpr int WPT = 4;
      u32 wnon = 0;
      bool wdone = false;
      u64 wv[WPT], wid[WPT];
      u64 whi = 0, ws = 0, we = 0;
      if (V == PIP_RP_FINAL && cursor >= 0) {
        whi = (u64)cursor;
        const u64 wlo = whi + 1 >= A.span_cap ? whi + 1 - A.span_cap : 0;
        part(whi - wlo + 1, G, b, ws, we);
        if (we - ws <= (u64)WPT * T) {
          wdone = true;
#pragma unroll
          for (int q = 0; q < WPT; ++q) {
            const u64 x = ws + tid + (u64)q * T;
            wid[q] = x < we ? whi - x : ~0ull;
            wv[q] = x < we ? __ldcs(A.h + wid[q]) : ~0ull;
          }
        }
      }
      auto mark_next = [&](u32 t) -> u32 {
        const u32 bit = 1u << (t & 31);
        if (atomicOr(Bp + (t >> 5), bit) & bit) {
          atomicOr(Cp + (t >> 5), bit);
          return 0u;
        }
        return 4u;
      };
      for (u64 k = s + tid; k < e; k += T) {
        const u32 tw = __ldcs(tg_n + k), i = __ldcs(ids_n + k);
        const u32 t = tw & RP_TMASK;
        if ((tw >> 31) && (t < dlo || t > dhi)) claims1 += 1;
        const u32 cw = __ldcg(Cc + (t >> 5)), bw = __ldcg(Bc + (i >> 5));
        // small grids (MB == 1, L2-resident a[]): both words of the swap
        // travel with the bitmap words, one L2 round trip less per round
        // (a committing iterate's words are touched by nobody else this round)
        u64 xs = 0, ys = 0;
        if (MB == 1 && PIP_RP_SPEC1) {
          xs = __ldcg(A.a + i);
          ys = __ldcg(A.a + t);
        }
        if ((cw >> (t & 31)) & 1u) {
          A.slot[k] = table_reserve(A.table, A.logcap, t, i, dclaim, &g->sync.error);
          A.cflag[k] = 2;
        } else {
          const bool c = !((bw >> (i & 31)) & 1u);
          if (c) {
            A.cflag[k] = 1;
            if (!(A.dbg & 1)) {
              if (MB == 1 && PIP_RP_SPEC1) {
                A.a[i] = ys;
                A.a[t] = xs;
              } else {
                rp_swap<BM>(A.a, i, t, A.dbg);
              }
            }
          } else {
            A.cflag[k] = (unsigned char)mark_next(t);
            fails += 1;
          }
        }
      }
      if (wdone) {
#pragma unroll
        for (int q = 0; q < WPT; ++q) wnon += wid[q] != ~0ull && wv[q] != wid[q];
      }
      {
        // claims (summed by the next retire) and the next window's count
        const u64 c = block_sum(((u64)wnon << 32) | claims1, s_red);
        if (tid == 0) {
          A.claimcnt[b] = (u32)c;
          if (wdone) A.wcnt[b] = (u32)(c >> 32);
        }
      }
      if (!grid_barrier(&g->sync, gen)) break;
      for (u64 k = s + tid; k < e; k += T) {
        if (__ldcs(A.cflag + k) != 2) continue;
        const u32 t = __ldcs(tg_n + k) & RP_TMASK, i = __ldcs(ids_n + k);
        const bool own = !((__ldcg(Bc + (i >> 5)) >> (i & 31)) & 1u);
        const u32 sl = __ldcg(A.slot + k);
        const u64 w = sl == RP_NOSLOT ? RP_EMPTY : __ldcg(A.table + sl);
        const bool c = own && w != RP_EMPTY && (u32)(w >> 32) == t && (u32)w == i;
        if (c) {
          A.cflag[k] = 1u | 8u;
          if (!(A.dbg & 1)) {  // PIP_RP_DBG=1: measurement only, no swaps
            rp_swap<BM>(A.a, i, t, A.dbg);
          }
        } else {
          A.cflag[k] = (unsigned char)(mark_next(t) | (sl == RP_NOSLOT ? 0u : 8u));
          fails += 1;
        }
      }
      const u64 f = block_sum(fails, s_red);
      if (tid == 0) A.failcnt[b] = (u32)f;
    } else if (BM == 2 || BM == 3) {
      // P3b: the iterates that found their target already marked (list lc)
      // reserve in a write-max table sized for them alone (L2-resident);
      // then every first marker looks its target up there: absent => it is
      // the only reserver and commits right away, present => it joins the
      // write-max and is resolved in the short P4 with the others (cflag 2).
      WSTAT_T0();
    if (!grid_barrier(&g->sync, gen)) break;
    WSTAT_T1(1);
      tick(2);
      u64 claims_total, dummy, lc_total, lc_before;
      if (BM == 2) {  // BM 3 counts distinct targets at the end of the round
        sum_counts(A.claimcnt, G, b, s_red, claims_total, dummy);
        RSET(if (claims_total > R.peak) R.peak = claims_total);
      }
      sum_counts(A.lccnt, G, b, s_red, lc_total, lc_before);
      u32 lg = 0;
      if (lc_total) {
        lg = 8;
        // load <= 1/4 (BM 2) or 1/2 (BM 3: the list is longer, the table
        // must stay in L2 next to the folded bitmap)
        while ((1ull << lg) < (u64)A.tload * lc_total) ++lg;
        if (lg > A.logcap) lg = A.logcap;
      }
      int c2 = 0;  // BM 3: listed claims of new targets - first markers that joined
      RSET(R.logcap_c = lg);
      u64 s, e;
      if (BM == 3) lpart(newF, nfail, A.wf, A.wn, G, b, s, e);
      else part(newF, G, b, s, e);
      u32 dclaim = 0;
      if (lc_total) {
        const u32 mine = __ldcg(A.lccnt + b);
        for (u32 q = tid; q < mine; q += T) {
          const u64 k = s + __ldcg(A.lc + s + q);
          const u32 t = __ldcs(tg_n + k);
          const u32 before = dclaim;
          table_reserve(A.table, lg, t, __ldcs(ids_n + k), dclaim, &g->sync.error);
          if (A.lf) atomicOr(A.lf + ((t & ((1u << RP_LF_LOG2) - 1u)) >> 5), 1u << (t & 31));
          if (BM == 3 && dclaim != before && (t < dlo || t > dhi)) c2 += 1;
        }
        WSTAT_T0();
    if (!grid_barrier(&g->sync, gen)) break;
    WSTAT_T1(2);
      }
      u32 fails = 0;
      // One item per thread per step (4 CTAs/SM of 64 registers beat 2 CTAs/SM
      // with 4-item batches: 110 vs 175 ms at 2^30; with the round state out
      // of the registers, 2 / 4 items per step with every wave of loads
      // issued for all items first: 142 / 179 ms at 4 CTAs per SM against
      // 128, 132 at 6 against 117 -- resident warps, not loads per thread,
      // are what this pass wants), but the step's loads are
      // issued in two waves instead of a chain: {cflag, target, id} of the
      // next item travel while this one finishes (software pipeline), and the
      // table probe and the own-check word go out together.
      auto commit_range = [&](const u64 s, const u64 e) {
      u64 k = s + tid;
      u32 ncf = 1, nt = 0, ni = 0;
      if (k < e) {
        ncf = __ldcs(A.cflag + k);
        nt = __ldcs(tg_n + k);
        ni = __ldcs(ids_n + k);
      }
      for (; k < e; k += T) {
        const u32 cf = ncf, t = nt, i = ni;
        if (k + T < e) {
          ncf = __ldcs(A.cflag + k + T);
          nt = __ldcs(tg_n + k + T);
          ni = __ldcs(ids_n + k + T);
        }
        if (cf) continue;
        const bool maybe = lc_total && (!A.lf || ((__ldcg(A.lf + ((t & ((1u << RP_LF_LOG2) - 1u)) >> 5)) >> (t & 31)) & 1u));
        const u64 w0 = maybe ? __ldcg(A.table + rp_home(t, lg)) : RP_EMPTY;
        const u32 bw = __ldcg(A.bmB + (i >> 5));
#if PIP_RP_XPRE
        // a[i] travels with the decision loads (ids are dense and descending,
        // so these reads are near-coalesced): a committing iterate's exchange
        // can leave as soon as the decision is made
        const u64 xpre = (BM == 3) ? __ldcg(A.a + i) : 0ull;
#endif
        u32 v;
        if (w0 != RP_EMPTY && ((u32)(w0 >> 32) == t || table_lookup(A.table, lg, t, v))) {
          table_reserve(A.table, lg, t, i, dclaim, &g->sync.error);
          A.cflag[k] = 2;
          if (BM == 3 && (t < dlo || t > dhi)) c2 -= 1;  // its target was counted as listed
          continue;
        }
        const bool c = !((bw >> (i & 31)) & 1u);
        A.cflag[k] = c;
        if (c) {
          if (!(A.dbg & 1)) {  // PIP_RP_DBG=1: measurement only, no swaps
#if PIP_RP_XPRE
            if (BM == 3 && !(A.dbg & 2u))
              A.a[i] = (u64)atomicExch((unsigned long long*)A.a + t, (unsigned long long)xpre);
            else
              rp_swap<BM>(A.a, i, t, A.dbg);
#else
            rp_swap<BM>(A.a, i, t, A.dbg);
#endif
          }
        } else {
          fails += 1;
        }
      }
      };
      // Scheme 3: the last RP_STEAL_PCT % of every part is not the part
      // owner's alone: it is cut into pieces of RP_STEAL_STEPS steps that
      // whichever CTA has finished its own share takes by ticket (round-robin
      // over the parts), so the CTAs reach the barrier together instead of
      // waiting ~9% of the pass for the slowest.  A piece lies inside one part;
      // its failures are added to that part's count (the next round's retire
      // packs by part).
      u64 ms = e;  // my part: [s, ms) mine, [ms, e) shared
      const bool steal = BM == 3 && A.steal_pct && G > 1;
      u64 plen = 0;
      if (steal) {
        // every part keeps the same shared length (parts differ by <= a few items)
        plen = (newF / G) * A.steal_pct / 100;
        plen -= plen % T;
        ms = e - s > plen ? e - plen : s;
      }
      {
        // one call site: first my own share, then pieces by ticket
        const u64 piece = (u64)RP_STEAL_STEPS * T;
        const u64 npieces = steal && plen ? ((plen + piece - 1) / piece) * G : 0;
        u64 lo = s, hi = ms;
        u32 own_fails = 0, pcur = b;
        bool mine = true;
        for (;;) {
          commit_range(lo, hi);
          if (!npieces) {
            own_fails = fails;
            break;
          }
          if (mine) {
            own_fails = fails;
            mine = false;
          } else {
            const u64 fp = block_sum(fails, s_red);
            if (tid == 0 && fp) atomicAdd(A.failcnt + pcur, (u32)fp);
          }
          fails = 0;
          __syncthreads();
          if (tid == 0) s_red[33] = atomicAdd((unsigned long long*)&g->ticket, 1ull);
          __syncthreads();
          const u64 tk = s_red[33];
          if (tk >= npieces) break;
          // tickets go round-robin over the parts (ticket -> piece is one-to-one)
          pcur = (u32)(tk % G);
          u64 ps, pe;
          lpart(newF, nfail, A.wf, A.wn, G, pcur, ps, pe);
          const u64 pms = pe - ps > plen ? pe - plen : ps;
          lo = pms + (tk / G) * piece;
          hi = lo + piece < pe ? lo + piece : pe;
          if (lo > hi) lo = hi;
        }
        fails = own_fails;
      }
      if (lc_total) {
        WSTAT_T0();
    if (!grid_barrier(&g->sync, gen)) break;
    WSTAT_T1(3);
        // P4: iterates on collided targets
        for (u64 k = s + tid; k < e; k += T) {
          if (__ldcs(A.cflag + k) != 2) continue;
          const u32 t = __ldcs(tg_n + k), i = __ldcs(ids_n + k);
          const bool own = !((__ldcg(A.bmB + (i >> 5)) >> (i & 31)) & 1u);
          u32 v = 0;
          const bool c = own && table_lookup(A.table, lg, t, v) && v == i;
          A.cflag[k] = c;
          if (c) {
            if (!(A.dbg & 1)) {
              rp_swap<BM>(A.a, i, t, A.dbg);
            }
          } else {
            fails += 1;
          }
        }
      }
      const u64 f = block_sum(fails, s_red);
      if (tid == 0) {
        if (BM == 3) atomicAdd(A.failcnt + b, (u32)f);  // zeroed in the mark phase; others may have added
        else A.failcnt[b] = (u32)f;
      }
      if (BM == 3) {
        const u64 c2s = block_sum((u64)(long long)c2, s_red);
        if (tid == 0) A.claim2[b] = (u32)c2s;
      }
    } else {
    if (!grid_barrier(&g->sync, gen)) break;
    tick(2);

    // ======================= P4: commit + swap ==============================
    {
      u64 claims_total, dummy;
      sum_counts(A.claimcnt, G, b, s_red, claims_total, dummy);
      RSET(if (claims_total > R.peak) R.peak = claims_total);
      u64 s, e;
      part(newF, G, b, s, e);
      u32 fails = 0;
      for (u64 k = s + tid; k < e; k += T) {
        const u32 i = __ldcs(ids_n + k), t = __ldcs(tg_n + k);
        bool own, tgt;
        u32 v = 0;
        if (V == PIP_RP_FINAL && k >= nfail) {
          const u32 dv = __ldcg(A.dense + (dhi - i));
          own = dv == 0 || dv == i + 1u;
        } else if (V == PIP_RP_NAIVE || V == PIP_RP_FLAT) {
          own = table_lookup(A.table, A.logcap, i, v) && v == i;
        } else {
          own = !table_lookup(A.table, A.logcap, i, v) || v == i;
        }
        if (V == PIP_RP_FINAL && t >= dlo && t <= dhi) {
          tgt = __ldcg(A.dense + (dhi - t)) == i + 1u;
        } else {
          const u32 sl = __ldcg(A.slot + k);
          const u64 w = sl == RP_NOSLOT ? RP_EMPTY : __ldcg(A.table + sl);
          tgt = w != RP_EMPTY && (u32)(w >> 32) == t && (u32)w == i;
        }
        const bool c = own && tgt;
        A.cflag[k] = c;
        if (c) {
          if (!(A.dbg & 1)) {  // PIP_RP_DBG=1: measurement only, no swaps
            rp_swap<BM>(A.a, i, t, A.dbg);
          }
        } else {
          fails += 1;
        }
      }
      const u64 f = block_sum(fails, s_red);
      if (tid == 0) A.failcnt[b] = (u32)f;
    }
    }
    RSET(R.fill = newF; R.nfail_prev = nfail; R.ping = nw; R.rounds += 1; R.first = 0; R.dlo = dlo;
         R.dhi = dhi; R.cursor = cursor; R.wpre = 0; R.rlo = band_lo; R.rhi = band_hi);
    bool wcounted = false;
    if (BM == 1) {  // P3b counted the next window when it fit its loads
      const u64 whi = cursor >= 0 ? (u64)cursor : 0;
      const u64 wlo = whi + 1 >= A.span_cap ? whi + 1 - A.span_cap : 0;
      u64 ws, we;
      part(whi - wlo + 1, G, b, ws, we);
      wcounted = cursor >= 0 && we - ws <= (u64)4 * T;
      if (wcounted) RSET(R.wpre = 1);
    }
    if (V == PIP_RP_FINAL && cursor >= 0 && !wcounted) {  // count the next round's window now
      hi = (u64)cursor;
      lo = hi + 1 >= A.span_cap ? hi + 1 - A.span_cap : 0;
      wd = hi - lo + 1;
      u64 ws, we;
      part(wd, G, b, ws, we);
      u64 c = we > ws ? count_nonself_range(A, hi - (we - 1), hi - ws) : 0;
      c = block_sum(c, s_red);
      if (tid == 0) A.wcnt[b] = (u32)c;
      RSET(R.wpre = 1);
    }
    WSTAT_T0();
    if (!grid_barrier(&g->sync, gen)) break;
    WSTAT_T1(4);
    tick(3);
    if (BM == 3) {
      // distinct out-of-window targets of the round (the reference table's
      // keys): first markers outside the window + listed targets no first
      // marker holds (listed claims - joined first markers)
      u64 fm, dummy;
      sum_counts(A.claimcnt, G, b, s_red, fm, dummy);
      const long long d = (long long)fm + sum_counts_signed(A.claim2, G, s_red);
      RSET(if (d > 0 && (u64)d > R.peak) R.peak = (u64)d);
    }
    if (A.progress && b == 0 && tid == 0) {
      // this round's list is descending (failures first, then the fresh
      // window), so its head bounds every pending id; every CTA's swaps
      // are ordered before the barrier above
      const u64 top = R.fill ? (u64)__ldcg(ids_n) : (R.cursor >= 0 ? (u64)R.cursor : 0);
      __threadfence_system();
      *(volatile u64*)A.progress = top;
    }
    if (++rounds_here >= A.rounds_limit) break;  // pause: host drains counts
  }
  if (b == 0 && tid == 0) {
    *A.resume = R;
    for (int i = 0; i < 4; ++i) g->t[i] += s_tacc[i];
  }
#if PIP_RP_WAITSTAT
  if (tid == 0)
    for (int i = 0; i < 5; ++i) atomicAdd((unsigned long long*)&g->wsum[i], (unsigned long long)wacc[i]);
#endif
}

// ---------------------------------------------------------------------------
// host

struct RpLayout {
  size_t ids[2], tg[2], slot, cflag, dense, table, failcnt, wcnt, claimcnt, rcounts, global,
      resume, vcnt, bmB, bmC, lc, lccnt, total;
  u64 bm_words;
  int bm;  // 0 table (+dense window), 1 bitmaps B and C, 2 bitmap B + collided lists,
          // 3 folded collision bitmap + own band of B + collided lists + H block counts
  size_t bmF, claim2, bcnt, lf;
  u32 logf;
};

static u64 pow2_at_least(u64 x) {
  u64 c = 8;  // ReservationTable.MIN_CAPACITY
  while (c < x) c <<= 1;
  return c;
}

static int rp_gmax() { return num_sms(current_device()) * 8; }

static RpLayout rp_layout_mode(u64 n, u64 prefix, int variant, u64 cap, int gmax, int bm) {
  RpLayout L{};
  L.bm = bm;
  size_t off = 0;
  auto take = [&](size_t bytes) {
    size_t o = off;
    off += (bytes + 255) & ~(size_t)255;
    return o;
  };
  L.ids[0] = take(prefix * 4);
  L.ids[1] = take(prefix * 4);
  L.tg[0] = take(prefix * 4);
  L.tg[1] = take(prefix * 4);
  L.slot = take(bm == 2 ? 0 : prefix * 4);
  L.cflag = take(prefix);
  L.dense = take(variant == PIP_RP_FINAL && !bm ? (prefix + prefix / 4 + 8) * 4 : 0);
  // BM 1: only the iterates on twice-hit targets use the table, at most
  // prefix / 2 distinct keys
  L.table = take((bm == 1 ? pow2_at_least(prefix) : cap) * 8);
  L.failcnt = take((size_t)gmax * 4);
  L.wcnt = take((size_t)gmax * 4);
  L.claimcnt = take((size_t)gmax * 4);
  L.rcounts = take(RP_ROUND_CHUNK * 8);
  L.global = take(sizeof(RpGlobal));
  L.resume = take(sizeof(RpResume));
  L.vcnt = take(16);  // (rcounts .. vcnt are read back by one copy)
  L.bm_words = bm ? (n + 31) / 32 : 0;
  L.bmB = take(L.bm_words * 4 * (bm == 1 ? 2 : 1));  // BM 1: one pair per round parity
  L.bmC = take(bm == 1 ? L.bm_words * 4 * 2 : 0);
  L.lc = take(bm >= 2 ? prefix * 4 : 0);
  L.lccnt = take(bm >= 2 ? (size_t)gmax * 4 : 0);
  L.logf = 0;
  if (bm == 3) {
    u32 lf = 10;
    while (lf < 28 && (1ull << lf) < n) ++lf;
    if (const char* e = getenv("PIP_RP_FOLD_LOG2")) lf = (u32)atoi(e) < 10 ? 10 : (u32)atoi(e);
    if (lf > 31) lf = 31;
    L.logf = lf;
  }
  L.bmF = take(bm == 3 ? (1ull << L.logf) / 8 : 0);
  L.claim2 = take(bm == 3 ? (size_t)gmax * 4 : 0);
  L.bcnt = take(bm == 3 ? ((n >> RP_BLK_SHIFT) + 1) * 4 : 0);
  L.lf = take(bm >= 2 ? (1ull << RP_LF_LOG2) / 8 : 0);
  L.total = off;
  return L;
}

static u64 rp_capacity(u64 prefix, int variant) {
  const bool two_res = variant == PIP_RP_NAIVE || variant == PIP_RP_FLAT;
  return pow2_at_least(two_res ? 4 * prefix : 2 * prefix);
}

// bitmap reservations for `final` whenever they fit the acceptance gate
// (workspace <= 8 b(n) words, test_acceptance.py:257).  Mode 1 (bitmaps B
// and C) while C is small enough to live in L2 (n <= 2^28: one phase less per
// round); mode 2 (B + collided lists, L2-resident per-round table) above
// that, where the random C reads would go to HBM.  PIP_RP_BM=0/1/2 forces.
static RpLayout rp_layout(u64 n, u64 prefix, int variant, u64 cap, int gmax) {
  if (variant == PIP_RP_FINAL) {
    int want = n < (1ull << 28) ? 1 : 3;  // measured crossover (2^27: 16.4 vs 18.2 ms, 2^28: 33.8 vs 32.0)
    if (const char* e = getenv("PIP_RP_BM")) want = atoi(e);
    if (want == 1 && n > (1ull << 31)) want = 3;  // BM 1 keeps a flag in target bit 31
    if (want >= 1 && want <= 3) {
      const RpLayout Lb = rp_layout_mode(n, prefix, variant, cap, gmax, want);
      if ((Lb.total + 7) / 8 <= 8 * prefix || getenv("PIP_RP_BM")) return Lb;
      for (int alt : {3, 2, 1}) {
        if (alt == want) continue;
        const RpLayout Lo = rp_layout_mode(n, prefix, variant, cap, gmax, alt);
        if ((Lo.total + 7) / 8 <= 8 * prefix) return Lo;
      }
    }
  }
  return rp_layout_mode(n, prefix, variant, cap, gmax, 0);
}

size_t rp_cluster_workspace_bytes(u64 n, u64 prefix);
bool rp_cluster_eligible(u64 n, u64 prefix, u64 span_cap, int* K_out);
int rp_cluster_run(u64* a, const u64* h, u64 n, u64 prefix, u64 span_cap, void* ws, size_t ws_bytes,
                   u64* counts_host, u64 rounds_cap, pip_rp_stats* S, cudaStream_t st, int K);

size_t rp_workspace_bytes(u64 n, u64 prefix, int variant) {
  if (prefix < 1 || variant < 0 || variant > 3) return 0;
  if (prefix > n && n > 0) prefix = n;
  size_t t = rp_layout(n, prefix, variant, rp_capacity(prefix, variant), rp_gmax()).total;
  if (variant == PIP_RP_FINAL) {  // the small-n cluster path (rp_cluster.cu) may run instead
    const size_t c = rp_cluster_workspace_bytes(n, prefix);
    if (c > t) t = c;
  }
  return t;
}

__global__ void rp_init_kernel(RpResume* r, RpResume r0, u32* g, u32 gwords, u32* failcnt, u32 gmax) {
  for (u32 x = threadIdx.x; x < gwords; x += blockDim.x) g[x] = 0u;
  for (u32 x = threadIdx.x; x < gmax; x += blockDim.x) failcnt[x] = 0u;
  if (threadIdx.x == 0) *r = r0;
}

template <int V, int BM = 0>
static int rp_run(RpArgs& A, int grid, cudaStream_t st) {
  auto k = rp_kernel<V, BM>;
  if (BM == 1 && PIP_RP_SMALL1 && grid <= num_sms(current_device())) k = rp_kernel<V, BM == 1 ? BM : 0, BM == 1 ? 1 : 4>;
  void* args[] = {&A};
  PIP_CUDA(cudaLaunchCooperativeKernel((const void*)k, dim3(grid), dim3(RP_THREADS), args, 0, st));
  return PIP_OK;
}

int validate_counts(const u64* h, u64 n, u64* nonself, u64* invalid, void* scratch16,
                    cudaStream_t st, u32* bcnt);

int rp_device(u64* a, const u64* h, u64 n, u64 prefix, int variant, int debug,
              u64* counts_host, u64 rounds_cap, u64* trace_dev, void* ws, size_t ws_bytes,
              pip_rp_stats* stats, cudaStream_t st, const RpProgress* prog) {
  if (variant < 0 || variant > 3 || prefix < 1) return PIP_ERR_INVALID_ARG;
  if (n >= 0xffffffffull) return PIP_ERR_UNSUPPORTED;
  pip_rp_stats S{};
  S.prefix = prefix;
  if (n == 0) {
    if (stats) *stats = S;
    return PIP_OK;
  }
  // the client sizes its table / dense window from `prefix` (relaxed.py:84-89)
  const u64 cap = rp_capacity(prefix, variant);
  if (cap > (1ull << 31)) return PIP_ERR_UNSUPPORTED;
  const int dev = current_device();
  const int gmax = rp_gmax();
  const RpLayout Lrun = rp_layout(n, prefix, variant, cap, gmax);
  const u64 tcap = Lrun.bm == 1 ? pow2_at_least(prefix) : cap;  // table slots allocated
  u32 logcap = 0;
  while ((1ull << logcap) < tcap) ++logcap;
  if (!ws || ws_bytes < Lrun.total) return PIP_ERR_OOM;
  char* w = (char*)ws;
  // validate H and count the non-self iterates (relaxed.py:233, :239).  The
  // counts stay on the device for the round kernel (it clamps the prefix and
  // refuses invalid H before touching a[]), so nothing waits for the host
  // between the validation and the launch; only the opt-in cluster path
  // needs them on the host first.
  const bool cluster_req = variant == PIP_RP_FINAL && !debug && !trace_dev && !prog &&
                           getenv("PIP_RP_CLUSTER") != nullptr;
  u64* vcnt = (u64*)(w + Lrun.vcnt);
  u64 n_iter = 0, invalid = 0;
  int vrc = validate_counts(h, n, cluster_req ? &n_iter : nullptr, &invalid, vcnt, st,
                            Lrun.bm == 3 ? (u32*)(w + Lrun.bcnt) : nullptr);
  if (vrc) return vrc;
  S.table_capacity = cap;
  if (cluster_req) {
    if (invalid) return PIP_ERR_INVALID_SWAPS;
    S.n_iterates = n_iter;
    if (n_iter == 0) {
      if (stats) *stats = S;
      return PIP_OK;
    }
  }
  // ... while run_rounds clamps the active prefix to n_iterates (detres.py:267)
  const u64 P = cluster_req ? (prefix < n_iter ? prefix : n_iter) : prefix;
  // small n: the whole round loop on one thread-block cluster (rp_cluster.cu)
  if (cluster_req) {
    int K = 0;
    const u64 span = prefix + prefix / 4 + 8;
    if (variant == PIP_RP_FINAL && !debug && !trace_dev && !prog && rp_cluster_eligible(n, P, span, &K)) {
      const int rc = rp_cluster_run(a, h, n, P, span, ws, ws_bytes, counts_host, rounds_cap, &S, st, K);
      if (rc != PIP_ERR_UNSUPPORTED) {
        S.table_capacity = cap;
        S.workspace_words = (rp_cluster_workspace_bytes(n, P) + 7) / 8;
        if (stats) *stats = S;
        return rc;
      }
    }
  }
  RpArgs A{};
  A.a = a;
  A.h = h;
  A.n = n;
  A.prefix = P;
  A.span_cap = prefix + prefix / 4 + 8;
  A.rounds_limit = RP_ROUND_CHUNK;
  A.logcap = logcap;
  A.debug = debug ? 1u : 0u;
  A.targeted_clean_ok = (variant == PIP_RP_FINAL || variant == PIP_RP_ONERES) ? 1u : 0u;
  for (int p = 0; p < 2; ++p) {
    A.ids[p] = (u32*)(w + Lrun.ids[p]);
    A.tg[p] = (u32*)(w + Lrun.tg[p]);
  }
  A.slot = (u32*)(w + Lrun.slot);
  A.cflag = (unsigned char*)(w + Lrun.cflag);
  A.dense = (u32*)(w + Lrun.dense);
  A.table = (u64*)(w + Lrun.table);
  A.failcnt = (u32*)(w + Lrun.failcnt);
  A.wcnt = (u32*)(w + Lrun.wcnt);
  A.claimcnt = (u32*)(w + Lrun.claimcnt);
  A.round_counts = (u64*)(w + Lrun.rcounts);
  A.progress = prog ? prog->dev : nullptr;
  A.trace = trace_dev;
  A.g = (RpGlobal*)(w + Lrun.global);
  A.resume = (RpResume*)(w + Lrun.resume);
  A.bm_words = Lrun.bm_words;
  A.bmB = Lrun.bm ? (u32*)(w + Lrun.bmB) : nullptr;
  A.bmC = Lrun.bm == 1 ? (u32*)(w + Lrun.bmC) : nullptr;
  A.lc = Lrun.bm >= 2 ? (u32*)(w + Lrun.lc) : nullptr;
  A.lccnt = Lrun.bm >= 2 ? (u32*)(w + Lrun.lccnt) : nullptr;
  A.bmF = Lrun.bm == 3 ? (u32*)(w + Lrun.bmF) : nullptr;
  A.logf = Lrun.logf;
  A.dbg = getenv("PIP_RP_DBG") ? (u32)atoi(getenv("PIP_RP_DBG")) : 0u;
  A.steal_pct = getenv("PIP_RP_STEAL") ? (u32)atoi(getenv("PIP_RP_STEAL")) : PIP_RP_STEAL_DEFAULT;
  if (A.steal_pct > 100) A.steal_pct = 100;
  A.wf = getenv("PIP_RP_WF") ? (u32)atoi(getenv("PIP_RP_WF")) : PIP_RP_WF_DEFAULT;
  A.wn = getenv("PIP_RP_WN") ? (u32)atoi(getenv("PIP_RP_WN")) : PIP_RP_WN_DEFAULT;
  if (A.wf < 1 || A.wf > 64 || A.wn < 1 || A.wn > 64) A.wf = A.wn = 1;
  A.tload = 4u;
  const bool use_lf = !(getenv("PIP_RP_LF") && atoi(getenv("PIP_RP_LF")) == 0);
  A.lf = Lrun.bm >= 2 && use_lf ? (u32*)(w + Lrun.lf) : nullptr;
  if (const char* e = getenv("PIP_RP_TLOAD")) A.tload = (u32)atoi(e) < 2 ? 2u : (u32)atoi(e);
  A.claim2 = Lrun.bm == 3 ? (u32*)(w + Lrun.claim2) : nullptr;
  A.bcnt = Lrun.bm == 3 ? (const u32*)(w + Lrun.bcnt) : nullptr;
  A.vcnt = cluster_req ? nullptr : vcnt;

  PIP_CUDA(cudaMemsetAsync(A.table, 0xff, tcap * 8, st));
  if (variant == PIP_RP_FINAL && !Lrun.bm) PIP_CUDA(cudaMemsetAsync(A.dense, 0, A.span_cap * 4, st));
  if (Lrun.bm) {
    PIP_CUDA(cudaMemsetAsync(A.bmB, 0, Lrun.bm_words * 4 * (Lrun.bm == 1 ? 2 : 1), st));
    if (Lrun.bm == 1) PIP_CUDA(cudaMemsetAsync(A.bmC, 0, Lrun.bm_words * 4 * 2, st));
    if (Lrun.bm == 3) PIP_CUDA(cudaMemsetAsync(A.bmF, 0, (1ull << Lrun.logf) / 8, st));
    if (Lrun.bm >= 2) PIP_CUDA(cudaMemsetAsync(w + Lrun.lf, 0, (1ull << RP_LF_LOG2) / 8, st));
  }
  RpResume R0{};
  R0.cursor = (long long)n - 1;
  R0.first = 1;
  R0.dlo = 1;
  R0.dhi = 0;
  R0.rlo = 1;
  R0.rhi = 0;
  // resume state, barrier / error words and fail counts set by one kernel
  // (parameters by value: no host staging, no sync)
  rp_init_kernel<<<1, 256, 0, st>>>(A.resume, R0, (u32*)A.g, (u32)(sizeof(RpGlobal) / 4), A.failcnt,
                                    (u32)gmax);
  PIP_CHECK_LAUNCH();

  // grid: enough CTAs to give every thread ~2 iterates, at most co-resident
  int per_sm = 0;
  const void* kp = variant == PIP_RP_FINAL ? (Lrun.bm == 1   ? (const void*)rp_kernel<PIP_RP_FINAL, 1>
                                                 : Lrun.bm == 2 ? (const void*)rp_kernel<PIP_RP_FINAL, 2>
                                                 : Lrun.bm == 3 ? (const void*)rp_kernel<PIP_RP_FINAL, 3>
                                                                : (const void*)rp_kernel<PIP_RP_FINAL, 0>)
                   : variant == PIP_RP_ONERES ? (const void*)rp_kernel<PIP_RP_ONERES, 0>
                   : variant == PIP_RP_FLAT ? (const void*)rp_kernel<PIP_RP_FLAT, 0>
                                             : (const void*)rp_kernel<PIP_RP_NAIVE, 0>;
  PIP_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kp, RP_THREADS, 0));
  if (per_sm < 1) return PIP_ERR_UNSUPPORTED;
  {
    // scheme 3 is compiled for PIP_RP_MINB3 CTAs per SM: its commit pass is
    // latency-bound and gains from every resident warp (C4: 130.6 ms at 4,
    // 121.2 at 5, 118.4 at 6, 120.5 at 8, where the other phases spill)
    const int cap = getenv("PIP_RP_PERSM") ? atoi(getenv("PIP_RP_PERSM"))
                                           : (Lrun.bm == 3 ? PIP_RP_MINB3 : 4);
    if (per_sm > cap && cap >= 1 && cap <= 8) per_sm = cap;
    if (per_sm > 8) per_sm = 8;
  }
  u64 grid = (u64)per_sm * num_sms(dev);
  // about one iterate per thread for small prefixes (measured: fewer, fuller
  // CTAs are slower — rounds are latency-bound per thread), full grid otherwise
  u64 ipt = 1;
  if (const char* e = getenv("PIP_RP_IPT")) ipt = (u64)atoll(e) > 0 ? (u64)atoll(e) : 1;
  const u64 want = (P + RP_THREADS * ipt - 1) / (RP_THREADS * ipt);
  if (grid > want) grid = want;
  if (grid < 1) grid = 1;

  u64 recorded = 0;
  RpResume R{};
  RpGlobal Gh{};
  std::vector<char> blob(Lrun.vcnt + 16 - Lrun.rcounts);
  for (;;) {
    int rc;
    switch (variant) {
      case PIP_RP_FINAL:
        rc = Lrun.bm == 1   ? rp_run<PIP_RP_FINAL, 1>(A, (int)grid, st)
             : Lrun.bm == 2 ? rp_run<PIP_RP_FINAL, 2>(A, (int)grid, st)
             : Lrun.bm == 3 ? rp_run<PIP_RP_FINAL, 3>(A, (int)grid, st)
                            : rp_run<PIP_RP_FINAL, 0>(A, (int)grid, st);
        break;
      case PIP_RP_ONERES: rc = rp_run<PIP_RP_ONERES>(A, (int)grid, st); break;
      case PIP_RP_FLAT: rc = rp_run<PIP_RP_FLAT>(A, (int)grid, st); break;
      default: rc = rp_run<PIP_RP_NAIVE>(A, (int)grid, st); break;
    }
    if (rc) return rc;
    if (prog) {  // hand the final suffix to the caller while the rounds run
      cudaError_t q;
      static const int poll_us = getenv("PIP_RP_POLL_US") ? atoi(getenv("PIP_RP_POLL_US")) : 50;
      while ((q = cudaStreamQuery(st)) == cudaErrorNotReady) {
        prog->hook(prog->ctx, *prog->host);
        if (poll_us > 0) std::this_thread::sleep_for(std::chrono::microseconds(poll_us));
      }
      if (q != cudaSuccess) PIP_CUDA(q);
    }
    // one copy brings back the round counts, the barrier / error words, the
    // resume state and the validation counts (adjacent in the workspace)
    PIP_CUDA(cudaMemcpyAsync(blob.data(), w + Lrun.rcounts, blob.size(), cudaMemcpyDeviceToHost, st));
    PIP_CUDA(cudaStreamSynchronize(st));
    memcpy(&R, blob.data() + (Lrun.resume - Lrun.rcounts), sizeof(R));
    memcpy(&Gh, blob.data() + (Lrun.global - Lrun.rcounts), sizeof(Gh));
    if (A.vcnt) {
      u64 vc[2];
      memcpy(vc, blob.data() + (Lrun.vcnt - Lrun.rcounts), 16);
      if (vc[1]) return PIP_ERR_INVALID_SWAPS;  // a[] untouched
      S.n_iterates = vc[0];
      if (vc[0] == 0) {
        if (stats) *stats = S;
        return PIP_OK;
      }
    }
    if (Gh.sync.abort) return PIP_ERR_STALLED;
    // counts are recorded in P1 of the following round: all rounds but the
    // last completed one are available (all of them once done)
    const u64 have = R.done ? R.rounds : (R.rounds ? R.rounds - 1 : 0);
    if (have > recorded && counts_host) {
      const u64* chunk = (const u64*)blob.data();
      for (u64 r = recorded; r < have; ++r)
        if (r < rounds_cap) counts_host[r] = chunk[r % RP_ROUND_CHUNK];
    }
    if (have > recorded) recorded = have;
    if (Gh.sync.error) {
      S.rounds = R.rounds;
      if (stats) *stats = S;
      return (int)Gh.sync.error;
    }
    if (R.done) break;
    // reset the barrier for the next launch
    PIP_CUDA(cudaMemsetAsync(&A.g->sync.bar_count, 0, 8, st));
  }
  if (timing_enabled())
    fprintf(stderr,
            "[pip rp] n=%llu prefix=%llu rounds=%llu grid=%llu  retire+clean+window %.3f ms | "
            "refill %.3f | reserve %.3f | commit+swap %.3f ms\n",
            (unsigned long long)n, (unsigned long long)P, (unsigned long long)R.rounds,
            (unsigned long long)grid, Gh.t[0] * 1e-6, Gh.t[1] * 1e-6, Gh.t[2] * 1e-6,
            Gh.t[3] * 1e-6);
#if PIP_RP_WAITSTAT
  if (timing_enabled())
    fprintf(stderr, "[pip rp] mean ms per CTA inside barriers: after refill %.3f | after marks %.3f | after listed "
            "reserve %.3f | before resolve %.3f | end of round %.3f\n",
            Gh.wsum[0] * 1e-6 / grid, Gh.wsum[1] * 1e-6 / grid, Gh.wsum[2] * 1e-6 / grid,
            Gh.wsum[3] * 1e-6 / grid, Gh.wsum[4] * 1e-6 / grid);
#endif
  S.rounds = R.rounds;
  S.total_committed = R.total_committed;
  S.peak_table_count = R.peak;
  S.table_capacity = cap;
  S.workspace_words = (Lrun.total + 7) / 8;
  S.rounds_recorded = recorded < rounds_cap ? recorded : rounds_cap;
  if (stats) *stats = S;
  return PIP_OK;
}

}  // namespace pip
