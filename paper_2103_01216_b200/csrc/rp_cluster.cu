// Random permutation for small n on ONE thread-block cluster (BASELINE
// configs[0]: n = 10^6, b(n) = 20,000 iterates, ~87 rounds).
//
// Same deterministic-reservation rounds as rp.cu (relaxed.py:64-251 on
// detres.py:256-307, `final` variant with the bitmap reservations): the
// active set of a round is the previous round's failures plus the next
// b - #failures non-self ids in descending order from the window
// [cursor - span_cap + 1, cursor] (relaxed.py:107-120); iterate i commits iff
// no active iterate targets i and i is the largest active id targeting H[i];
// so rounds, committed-per-round and the table load are the reference's.
//
// Why a cluster: at this size a round is a chain of short dependent steps,
// and rp.cu pays a grid-wide barrier (~2 us of global atomics and polls)
// between them — 20 us per round.  Here the whole state lives in the
// distributed shared memory of a 16-CTA cluster (non-portable size; 8 when
// 16 is unavailable): the two reservation bitmaps B ("targeted") and C
// ("targeted twice") are striped over the CTAs' shared memory and set with
// DSMEM atomics, each CTA keeps its part of the active list locally, the
// window's H values are cached in shared memory between the count and the
// refill, and the phases are separated by hardware cluster barriers
// (barrier.cluster, ~0.2 us).  Only a, H and the rarely used write-max table
// (targets hit at least twice) live in global memory (L2-resident at this n).
//
// A round = 4 cluster barriers:
//   E/A  (end of the previous round) failures packed locally in order,
//        next window counted and its H values cached, counts published;
//   B    bitmaps and touched table slots cleared, fresh ids assigned to
//        CTAs (each tops its list up to ceil(b/K)), scattered by DSMEM;
//   C    marks: atomicOr B[t]; second markers set C[t]; distinct targets
//        outside the fresh window counted (peak_table_load);
//   D    C targets reserve in the write-max table; every other iterate
//        commits iff !B[i] and swaps a[i], a[t];
//   E    C-target iterates commit iff !B[i] and they hold the table's max.
// The order inside the active list differs from the reference's (failures
// stay in their CTA), which only the trace would show: calls that want a
// trace (or debug sweeps) use rp.cu.
#include <cooperative_groups.h>
#include <cstdio>
#include <cstdlib>
#include "common.cuh"

namespace cg = cooperative_groups;

namespace pip {

bool timing_enabled();

static constexpr int RC_THREADS = 1024;
static constexpr int RC_MAXK = 16;
static constexpr u64 RC_EMPTY = ~0ull;
static constexpr u32 RC_NOSLOT = 0xffffffffu;
static constexpr u32 RC_SELF = 0xffffffffu;

struct RcArgs {
  u64* a;
  const u64* h;
  u64 n, prefix, span_cap;
  u64* table;
  u32 logcap, wc_words, cap, part_cap;
  u64* round_counts;
  u64 rounds_cap;
  u64* out;  // [0] rounds [1] total committed [2] peak distinct targets [3] status
             // [4..8] ns per phase (CTA 0): B refill, C marks, D commits, E resolve, A pack+count
};

// published values, written into every CTA's copy by DSMEM stores; the
// end-of-round ones are double-buffered by round parity, so a round needs no
// barrier just to protect readers of the previous values
struct RcPub {
  u32 nfail[2][RC_MAXK], wcnt[2][RC_MAXK], fails[2][RC_MAXK], claims[RC_MAXK];
  u64 dlo, dhi;
};

__device__ __forceinline__ u64 rc_home(u32 key, u32 logcap) { return ((u64)key * GOLDEN) >> (64 - logcap); }

__device__ __forceinline__ u32 rc_reserve(u64* table, u32 logcap, u32 key, u32 val, u64* status) {
  const u64 mask = (1ull << logcap) - 1;
  u64 s = rc_home(key, logcap);
  const u64 want = ((u64)key << 32) | val;
  for (u64 step = 0; step <= mask; ++step) {
    u64 cur = __ldcg(table + s);
    if (cur == RC_EMPTY) {
      const u64 prev = atomicCAS(reinterpret_cast<unsigned long long*>(table + s), RC_EMPTY, want);
      if (prev == RC_EMPTY) return (u32)s;
      cur = prev;
    }
    if ((u32)(cur >> 32) == key) {
      if ((u32)cur < val) atomicMax(reinterpret_cast<unsigned long long*>(table + s), want);
      return (u32)s;
    }
    s = (s + 1) & mask;
  }
  atomicExch(reinterpret_cast<unsigned long long*>(status), (unsigned long long)PIP_ERR_TABLE);
  return RC_NOSLOT;
}

// block-wide exclusive rank of flag f in thread order; *tot = set flags
__device__ __forceinline__ u32 rc_rank(bool f, u32* s_w, u32* tot) {
  const u32 lane = lane_id(), warp = warp_id();
  const u32 m = __ballot_sync(0xffffffffu, f);
  if (lane == 0) s_w[warp] = __popc(m);
  __syncthreads();
  if (warp == 0) {
    const u32 v = s_w[lane];  // 32 warps of 32 threads
    u32 inc = v;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const u32 t = __shfl_up_sync(0xffffffffu, inc, o);
      if (lane >= (u32)o) inc += t;
    }
    s_w[lane] = inc - v;
    if (lane == 31) s_w[32] = inc;
  }
  __syncthreads();
  const u32 r = s_w[warp] + __popc(m & ((1u << lane) - 1u));
  *tot = s_w[32];
  __syncthreads();
  return r;
}

__device__ __forceinline__ u32 rc_block_sum(u32 v, u32* s_w) {
  v = __reduce_add_sync(0xffffffffu, v);
  if (lane_id() == 0) s_w[warp_id()] = v;
  __syncthreads();
  if (warp_id() == 0) {
    u32 x = __reduce_add_sync(0xffffffffu, s_w[lane_id()]);
    if (lane_id() == 0) s_w[33] = x;
  }
  __syncthreads();
  const u32 r = s_w[33];
  __syncthreads();
  return r;
}

template <int K>
__global__ void __launch_bounds__(RC_THREADS, 1) rp_cluster_kernel(RcArgs A) {
  extern __shared__ __align__(16) u32 sm[];
  __shared__ RcPub pub;
  __shared__ u32 s_w[40];
  cg::cluster_group cl = cg::this_cluster();
  const u32 me = cl.block_rank(), tid = threadIdx.x, T = blockDim.x;
  const u32 WC = A.wc_words, CAP = A.cap, PC = A.part_cap;
  u32* bB = sm;
  u32* bC = bB + WC;
  u32* ids = bC + WC;   // my part of the active list: failures first, then fresh ids
  u32* tg = ids + CAP;
  u32* slot = tg + CAP;  // table slot of a C-target reservation
  u32* hv = slot + CAP;  // cached window part: H value or RC_SELF
  unsigned char* cflag = (unsigned char*)(hv + PC);
  const u64 n = A.n, P = A.prefix, W = A.span_cap;

  for (u32 x = tid; x < WC; x += T) bB[x] = bC[x] = 0u;
  for (u32 x = tid; x < CAP; x += T) slot[x] = RC_NOSLOT;

  long long cursor = (long long)n - 1;
  u64 lo = 0, hi = 0, wd = 0, ps = 0, pe = 0;
  // count the non-self ids of my part of the window at `cursor` and cache H
  auto count_window = [&]() -> u32 {
    hi = (u64)cursor;
    lo = hi + 1 >= W ? hi + 1 - W : 0;
    wd = hi - lo + 1;
    ps = wd * me / K;
    pe = wd * (me + 1) / K;
    u32 c = 0;
    for (u64 q = ps + tid; q < pe; q += T) {
      const u64 id = hi - q;
      const u64 v = __ldcg(A.h + id);
      hv[q - ps] = v != id ? (u32)v : RC_SELF;
      c += v != id;
    }
    return rc_block_sum(c, s_w);
  };
  auto publish = [&](u32* field, u32 v) {  // field is a member of pub
    if (tid < K) *cl.map_shared_rank(field + me, tid) = v;
  };

  u32 ncur = 0, nfail_me = 0;
  u64 rounds = 0, total = 0, peak = 0, zero_rounds = 0;
  const bool tm = me == 0 && tid == 0;
  u64 tacc[5] = {0, 0, 0, 0, 0};
  u64 tlast = tm ? globaltimer_ns() : 0;
  auto tick = [&](int ph) {
    if (tm) {
      const u64 now = globaltimer_ns();
      tacc[ph] += now - tlast;
      tlast = now;
    }
  };
  u32 wc0 = cursor >= 0 ? count_window() : 0;
  publish(pub.nfail[0], 0u);
  publish(pub.wcnt[0], wc0);
  cl.sync();

  for (;;) {
    const u32 par = (u32)(rounds & 1);
    // ============ B: clear, refill ============
    for (u32 x = tid; x < WC; x += T) bB[x] = bC[x] = 0u;
    for (u32 k = tid; k < ncur; k += T) {
      const u32 s = slot[k];
      if (s != RC_NOSLOT) {
        A.table[s] = RC_EMPTY;
        slot[k] = RC_NOSLOT;
      }
    }
    __shared__ u32 nf[RC_MAXK], q[RC_MAXK], Q[RC_MAXK];
    u64 nfail = 0;
#pragma unroll
    for (int c = 0; c < K; ++c) nfail += pub.nfail[par][c];
    const u64 count = P - nfail;
    bool win = count > 0 && cursor >= 0;
    u64 wt = 0;
    while (win) {
      wt = 0;
#pragma unroll
      for (int c = 0; c < K; ++c) wt += pub.wcnt[par][c];
      if (wt > 0) break;
      cursor = (long long)lo - 1;  // empty window: move on (relaxed.py:119)
      win = cursor >= 0;
      const u32 wc = win ? count_window() : 0;
      cl.sync();  // everyone has read the old counts
      publish(pub.wcnt[par], wc);
      cl.sync();
    }
    const u64 fresh = win ? (count < wt ? count : wt) : 0;
    // quotas: CTA c tops its list up to CAP, in CTA order
    if (tid == 0) {
      u64 rem = fresh, run = 0;
      for (int c = 0; c < K; ++c) {
        nf[c] = pub.nfail[par][c];
        const u64 room = CAP > nf[c] ? CAP - nf[c] : 0;
        const u64 take = room < rem ? room : rem;
        q[c] = (u32)take;
        Q[c] = (u32)run;
        run += take;
        rem -= take;
      }
    }
    __syncthreads();
    if (fresh > 0) {
      u64 rbase = 0;
      for (u32 c = 0; c < me; ++c) rbase += pub.wcnt[par][c];
      const u64 np = pe - ps;
      u64 run = rbase;
      for (u64 q0 = 0; q0 < np && run < fresh; q0 += T) {
        const u64 k = q0 + tid;
        const u32 v = k < np ? hv[k] : RC_SELF;
        u32 tot;
        const u64 r = run + rc_rank(v != RC_SELF, s_w, &tot);
        if (v != RC_SELF && r < fresh) {
          const u32 id = (u32)(hi - (ps + k));
          int d = 0;  // the CTA whose quota holds rank r
          for (int c = 1; c < K; ++c)
            if (r >= Q[c] && q[c]) d = c;
          const u32 pos = nf[d] + (u32)(r - Q[d]);
          *cl.map_shared_rank(ids + pos, d) = id;
          *cl.map_shared_rank(tg + pos, d) = v;
          if (r == 0)
            for (int c = 0; c < K; ++c) *cl.map_shared_rank(&pub.dhi, c) = id;
          if (r == fresh - 1)
            for (int c = 0; c < K; ++c) *cl.map_shared_rank(&pub.dlo, c) = id;
        }
        run += tot;
      }
    } else if (tid < K) {
      *cl.map_shared_rank(&pub.dlo, tid) = 1;
      *cl.map_shared_rank(&pub.dhi, tid) = 0;
    }
    const u64 newF = nfail + fresh;
    if (newF == 0) break;  // every CTA sees the same counts
    const u32 nmine = nfail_me + q[me];
    cl.sync();
    tick(0);

    // ============ C: marks ============
    const u64 dlo = pub.dlo, dhi = pub.dhi;
    if (fresh > 0) cursor = (long long)dlo - 1;
    u32 claims = 0;
    for (u32 k = tid; k < nmine; k += T) {
      const u32 t = tg[k];
      const u32 w = t >> 5, bit = 1u << (t & 31);
      const u32 own = w / WC, lw = w % WC;
      const u32 old = atomicOr(cl.map_shared_rank(bB + lw, own), bit);
      if (old & bit) atomicOr(cl.map_shared_rank(bC + lw, own), bit);
      else if (t < dlo || t > dhi) claims += 1;
    }
    publish(pub.claims, rc_block_sum(claims, s_w));
    cl.sync();
    tick(1);

    // ============ D: commits on single-reserver targets; C targets reserve ============
    {
      u64 d = 0;
#pragma unroll
      for (int c = 0; c < K; ++c) d += pub.claims[c];
      if (d > peak) peak = d;
    }
    u32 fails = 0;
    for (u32 k = tid; k < nmine; k += T) {
      const u32 t = tg[k], i = ids[k];
      const u32 wt_ = t >> 5, bt = 1u << (t & 31), wi = i >> 5;
      // both DSMEM words travel together
      const u32 cword = *cl.map_shared_rank(bC + wt_ % WC, wt_ / WC);
      const u32 bword = *cl.map_shared_rank(bB + wi % WC, wi / WC);
      if (cword & bt) {
        slot[k] = rc_reserve(A.table, A.logcap, t, i, A.out + 3);
        cflag[k] = 2;
        continue;
      }
      const bool own = !((bword >> (i & 31)) & 1u);
      cflag[k] = own;
      if (own) {
        const u64 x = __ldcg(A.a + i), y = __ldcg(A.a + t);
        A.a[i] = y;
        A.a[t] = x;
      } else {
        fails += 1;
      }
    }
    cl.sync();
    tick(2);

    // ============ E: C targets resolve ============
    for (u32 k = tid; k < nmine; k += T) {
      if (cflag[k] != 2) continue;
      const u32 t = tg[k], i = ids[k];
      const u32 wi = i >> 5;
      const bool own = !((*cl.map_shared_rank(bB + wi % WC, wi / WC) >> (i & 31)) & 1u);
      const u32 s = slot[k];
      const u64 w = s == RC_NOSLOT ? RC_EMPTY : __ldcg(A.table + s);
      const bool c = own && w != RC_EMPTY && (u32)(w >> 32) == t && (u32)w == i;
      cflag[k] = c;
      if (c) {
        const u64 x = __ldcg(A.a + i), y = __ldcg(A.a + t);
        A.a[i] = y;
        A.a[t] = x;
      } else {
        fails += 1;
      }
    }
    // ---- A of the next round: pack my failures (in order), count the next window
    __syncthreads();
    tick(3);
    {
      u32 nf2 = 0;
      for (u32 k0 = 0; k0 < nmine; k0 += T) {
        const u32 k = k0 + tid;
        const bool f = k < nmine && cflag[k] == 0;
        u32 tot;
        const u32 r = rc_rank(f, s_w, &tot);
        u32 iv = 0, tv = 0;
        if (f) {
          iv = ids[k];
          tv = tg[k];
        }
        __syncthreads();  // reads of this chunk before the in-place writes
        if (f) {
          ids[nf2 + r] = iv;
          tg[nf2 + r] = tv;
        }
        nf2 += tot;
        __syncthreads();
      }
      nfail_me = nf2;
    }
    const u32 fsum = rc_block_sum(fails, s_w);
    const u32 wc = cursor >= 0 ? count_window() : 0;
    const u32 nx = par ^ 1u;  // last read two rounds ago: no barrier needed before the stores
    publish(pub.fails[nx], fsum);
    publish(pub.nfail[nx], nfail_me);
    publish(pub.wcnt[nx], wc);
    cl.sync();
    tick(4);
    u64 tf = 0;
#pragma unroll
    for (int c = 0; c < K; ++c) tf += pub.fails[nx][c];
    const u64 ncommit = newF - tf;
    if (me == 0 && tid == 0 && rounds < A.rounds_cap) A.round_counts[rounds] = ncommit;
    rounds += 1;
    total += ncommit;
    if (ncommit == 0) {
      if (++zero_rounds >= 64) {
        if (me == 0 && tid == 0) A.out[3] = PIP_ERR_LIVELOCK;
        break;
      }
    } else {
      zero_rounds = 0;
    }
    ncur = nmine;
  }
  cl.sync();  // no CTA leaves while others may still address its shared memory
  if (me == 0 && tid == 0) {
    A.out[0] = rounds;
    A.out[1] = total;
    A.out[2] = peak;
    for (int i = 0; i < 5; ++i) A.out[4 + i] = tacc[i];
  }
}

// ---------------------------------------------------------------------------
// host

struct RcPlan {
  int K;
  u32 wc_words, cap, part_cap;
  size_t smem;
};

static RcPlan rc_plan(u64 n, u64 P, u64 span, int K) {
  RcPlan p{};
  p.K = K;
  const u64 words = (n + 31) / 32;
  p.wc_words = (u32)((words + K - 1) / K);
  p.cap = (u32)((P + K - 1) / K);
  p.part_cap = (u32)((span + K - 1) / K + 1);
  p.smem = (size_t)(2 * p.wc_words + 3 * (size_t)p.cap + p.part_cap) * 4 + p.cap + 16;
  return p;
}

// workspace words (beyond the caller's a, h): table + round counts + out
size_t rp_cluster_workspace_bytes(u64 n, u64 prefix) {
  u64 cap = 8;
  while (cap < 2 * prefix) cap <<= 1;
  const u64 rcap = 4 * (n / (prefix ? prefix : 1)) + 4096;
  return (size_t)(cap * 8 + rcap * 8 + 128);
}

// eligible: final variant, no trace / debug, state fits the cluster's smem
bool rp_cluster_eligible(u64 n, u64 prefix, u64 span_cap, int* K_out) {
  // measured at C0 (n = 10^6): 1.80 ms against 1.76 ms for rp.cu's grid
  // kernel — the DSMEM atomics and reads cost as much as the grid barriers
  // they replace — so the cluster path is opt-in (PIP_RP_CLUSTER=1|8)
  const char* e = getenv("PIP_RP_CLUSTER");
  if (!e) return false;
  if (n < 2 || n > (1ull << 23) || prefix > 65536 || n / prefix > 65536) return false;
  int dev = current_device();
  int max_smem = 0;
  cudaDeviceGetAttribute(&max_smem, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev);
  const int want = e ? atoi(e) : 0;  // opt-in: 1 (16 CTAs, else 8) or 8
  if (want != 1 && want != 8 && want != 2) return false;
  for (int K : {16, 8}) {
    if (want == 8 && K == 16) continue;
    const RcPlan p = rc_plan(n, prefix, span_cap, K);
    if (p.smem + sizeof(RcPub) + 256 <= (size_t)max_smem) {
      *K_out = K;
      return true;
    }
  }
  return false;
}

template <int K>
static int rc_launch(const RcArgs& A, size_t smem, cudaStream_t st) {
  auto k = rp_cluster_kernel<K>;
  PIP_CUDA(cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  if (K > 8) PIP_CUDA(cudaFuncSetAttribute(k, cudaFuncAttributeNonPortableClusterSizeAllowed, 1));
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(K);
  cfg.blockDim = dim3(RC_THREADS);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeClusterDimension;
  at[0].val.clusterDim.x = K;
  at[0].val.clusterDim.y = 1;
  at[0].val.clusterDim.z = 1;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  PIP_CUDA(cudaLaunchKernelEx(&cfg, k, A));
  return PIP_OK;
}

// runs every round; returns PIP_ERR_UNSUPPORTED (nothing touched) when the
// cluster cannot be launched, so the caller falls back to rp.cu
int rp_cluster_run(u64* a, const u64* h, u64 n, u64 prefix, u64 span_cap, void* ws, size_t ws_bytes,
                   u64* counts_host, u64 rounds_cap, pip_rp_stats* S, cudaStream_t st, int K) {
  u64 cap = 8;
  u32 logcap = 3;
  while (cap < 2 * prefix) {
    cap <<= 1;
    ++logcap;
  }
  // round counts: as many as the workspace holds after the table (at least
  // 4 n / b + 4096 when sized by pip_rp_workspace_bytes); a longer run keeps
  // the first ones (rounds_recorded tells)
  if (!ws || ws_bytes < cap * 8 + 128 + 4096 * 8) return PIP_ERR_OOM;
  const u64 rcap = (ws_bytes - cap * 8 - 128) / 8;
  RcArgs A{};
  A.a = a;
  A.h = h;
  A.n = n;
  A.prefix = prefix;
  A.span_cap = span_cap;
  A.table = (u64*)ws;
  A.logcap = logcap;
  A.round_counts = A.table + cap;
  A.rounds_cap = rcap;
  A.out = A.round_counts + rcap;
  const RcPlan p = rc_plan(n, prefix, A.span_cap, K);
  A.wc_words = p.wc_words;
  A.cap = p.cap;
  A.part_cap = p.part_cap;
  PIP_CUDA(cudaMemsetAsync(A.table, 0xff, cap * 8, st));
  PIP_CUDA(cudaMemsetAsync(A.out, 0, 128, st));
  int rc = K == 16 ? rc_launch<16>(A, p.smem, st) : rc_launch<8>(A, p.smem, st);
  if (rc) {
    const cudaError_t e = cudaGetLastError();
    if (timing_enabled())
      fprintf(stderr, "[pip rp] cluster launch (K=%d, smem %zu) failed: %s; grid kernel instead\n", K,
              p.smem, cudaGetErrorString(e));
    if (getenv("PIP_RP_CLUSTER") && atoi(getenv("PIP_RP_CLUSTER")) == 2) return PIP_ERR_CUDA;
    return PIP_ERR_UNSUPPORTED;
  }
  u64 out[9];
  PIP_CUDA(cudaMemcpyAsync(out, A.out, sizeof(out), cudaMemcpyDeviceToHost, st));
  PIP_CUDA(cudaStreamSynchronize(st));
  const u64 rounds = out[0];
  u64 rec = rounds < rounds_cap ? rounds : rounds_cap;
  if (rec > rcap) rec = rcap;
  if (counts_host && rec) PIP_CUDA(cudaMemcpy(counts_host, A.round_counts, rec * 8, cudaMemcpyDeviceToHost));
  if (timing_enabled())
    fprintf(stderr, "[pip rp] cluster path: K=%d CTAs x %d threads, smem %zu B, %llu rounds | "
            "refill %.3f marks %.3f commit %.3f resolve %.3f pack+count %.3f ms\n", K, RC_THREADS,
            p.smem, (unsigned long long)rounds, out[4] * 1e-6, out[5] * 1e-6, out[6] * 1e-6,
            out[7] * 1e-6, out[8] * 1e-6);
  S->rounds = rounds;
  S->total_committed = out[1];
  S->peak_table_count = out[2];
  S->rounds_recorded = rec;
  if (out[3]) return (int)out[3];
  return PIP_OK;
}

}  // namespace pip
