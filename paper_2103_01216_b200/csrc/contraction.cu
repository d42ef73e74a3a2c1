// List contraction and list ranking on deterministic-reservation rounds
// (contraction.list_contract / list_rank, contraction.py:168-365, driven by
// detres.run_rounds, detres.py:256-307).
//
// Round structure identical to the reference (so rounds, committed-per-round
// and the per-round committed sets match): the active prefix holds the
// failures of the previous round in order, then fresh ids ascending from a
// cursor, up to b(n) iterates.  An active element commits iff its priority
// is below that of every neighbour that is itself active (pending and below
// the cursor — every issued id that is not spliced is in the prefix, and
// live links only point at live elements); committed elements splice out.
// Adjacent elements cannot both commit (distinct priorities), so the splices
// of a round touch disjoint slots and run in parallel.
//
// Per round (host loop, one sync for the round's commit count):
//   K1 eligibility (+ fresh ids written into the prefix)
//   K2 splice      (plain: neighbours re-linked, v keeps (u, x);
//                   weighted: prev packs (pointer << 32 | incoming distance),
//                   v keeps (parent, distance))
//   K3 pack        stable compaction of the failures (block counts, one-CTA
//                  scan, scatter into the other ids buffer)
// Ranking then resolves rank(v) = dist(v) + rank(parent) in dependence waves
// over the contraction forest (contraction.py:292-320): a node is final once
// its parent is (in place: the DONE mark replaces the parent pointer).
#include <cstdio>
#include <vector>
#include "sync.cuh"

namespace pip {

static constexpr u64 LC_NIL = ~0ull;
static constexpr u64 LC_DONE = ~0ull - 1;  // ranking: "rank final" (contraction.py:44)
static constexpr u32 LC_NIL32 = 0xffffffffu;
static constexpr int LC_T = 256;
static constexpr int LC_BLK = 1024;  // items per compaction block

struct LcDev {
  u64 ncommit;
  u64 pending, ready;
};

template <bool RANK>
__global__ void __launch_bounds__(LC_T) lc_elig_kernel(const u64* __restrict__ nxt,
                                                       const u64* __restrict__ prv,
                                                       const u64* __restrict__ p, u32* ids,
                                                       unsigned char* cflag, u64 fill, u64 nfail,
                                                       u64 cursor0, u64 cursor1) {
  for (u64 k = (u64)blockIdx.x * LC_T + threadIdx.x; k < fill; k += (u64)gridDim.x * LC_T) {
    u32 v;
    if (k < nfail) {
      v = ids[k];
    } else {
      v = (u32)(cursor0 + (k - nfail));
      ids[k] = v;
    }
    const u64 x = nxt[v];
    const u64 pu = prv[v];
    const u64 u = RANK ? ((pu >> 32) == LC_NIL32 ? LC_NIL : (pu >> 32)) : pu;
    const u64 pv = p[v];
    bool e = true;
    if (x != LC_NIL && x < cursor1) e = e && pv < p[x];
    if (u != LC_NIL && u < cursor1) e = e && pv < p[u];
    cflag[k] = e ? 1 : 0;
  }
}

template <bool RANK>
__global__ void __launch_bounds__(LC_T) lc_splice_kernel(u64* nxt, u64* prv, const u32* __restrict__ ids,
                                                         const unsigned char* __restrict__ cflag,
                                                         u64 fill, LcDev* d) {
  u32 c = 0;
  for (u64 k = (u64)blockIdx.x * LC_T + threadIdx.x; k < fill; k += (u64)gridDim.x * LC_T) {
    if (!cflag[k]) continue;
    ++c;
    const u32 v = ids[k];
    const u64 x = nxt[v];
    if (!RANK) {
      const u64 u = prv[v];
      if (u != LC_NIL) nxt[u] = x;
      if (x != LC_NIL) prv[x] = u;
    } else {
      const u64 packed = prv[v];
      const u64 u = packed >> 32, w_uv = packed & LC_NIL32;
      if (x != LC_NIL) {
        const u64 w_vx = prv[x] & LC_NIL32;
        prv[x] = (u << 32) | (w_uv + w_vx);
      }
      if (u != LC_NIL32) nxt[u] = x;
      nxt[v] = u != LC_NIL32 ? u : LC_NIL;  // dead slots: (parent, distance to it)
      prv[v] = w_uv;
    }
  }
  c = __reduce_add_sync(0xffffffffu, c);
  if ((threadIdx.x & 31) == 0 && c) atomicAdd((unsigned long long*)&d->ncommit, (unsigned long long)c);
}

// failures per block of LC_BLK items
__global__ void __launch_bounds__(LC_T) lc_count_kernel(const unsigned char* __restrict__ cflag, u64 fill,
                                                        u32* bcnt) {
  const u64 b0 = (u64)blockIdx.x * LC_BLK;
  u32 c = 0;
  for (u32 i = threadIdx.x; i < LC_BLK; i += LC_T)
    if (b0 + i < fill) c += cflag[b0 + i] == 0;
  __shared__ u32 s_w[LC_T / 32];
  c = __reduce_add_sync(0xffffffffu, c);
  if ((threadIdx.x & 31) == 0) s_w[threadIdx.x >> 5] = c;
  __syncthreads();
  if (threadIdx.x == 0) {
    u32 t = 0;
    for (int w = 0; w < LC_T / 32; ++w) t += s_w[w];
    bcnt[blockIdx.x] = t;
  }
}

// exclusive scan of the block counts (one CTA)
__global__ void __launch_bounds__(1024) lc_scan_kernel(u32* bcnt, u64 nblk) {
  __shared__ u32 s[1024];
  u32 carry = 0;
  for (u64 c0 = 0; c0 < nblk; c0 += 1024) {
    const u64 i = c0 + threadIdx.x;
    const u32 v = i < nblk ? bcnt[i] : 0u;
    s[threadIdx.x] = v;
    __syncthreads();
    for (u32 o = 1; o < 1024; o <<= 1) {
      const u32 y = threadIdx.x >= o ? s[threadIdx.x - o] : 0u;
      __syncthreads();
      s[threadIdx.x] += y;
      __syncthreads();
    }
    if (i < nblk) bcnt[i] = carry + s[threadIdx.x] - v;
    carry += s[1023];
    __syncthreads();
  }
}

// stable scatter of the failures (block-local order by a warp-ballot scan)
__global__ void __launch_bounds__(LC_T) lc_pack_kernel(const u32* __restrict__ ids_in,
                                                       const unsigned char* __restrict__ cflag, u64 fill,
                                                       const u32* __restrict__ bbase, u32* ids_out) {
  const u64 b0 = (u64)blockIdx.x * LC_BLK;
  __shared__ u32 s_w[LC_T / 32];
  const u32 lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  u32 base = bbase[blockIdx.x];
  for (u32 c0 = 0; c0 < LC_BLK; c0 += LC_T) {
    const u64 k = b0 + c0 + threadIdx.x;
    const bool f = k < fill && cflag[k] == 0;
    const unsigned bal = __ballot_sync(0xffffffffu, f);
    if (lane == 0) s_w[w] = __popc(bal);
    __syncthreads();
    u32 before = 0, tot = 0;
    for (u32 i = 0; i < LC_T / 32; ++i) {
      before += i < w ? s_w[i] : 0u;
      tot += s_w[i];
    }
    if (f) ids_out[base + before + __popc(bal & ((1u << lane) - 1u))] = ids_in[k];
    base += tot;
    __syncthreads();
  }
}

// list_rank's packing of prev (contraction.py:344-347): (prev << 32 | 1),
// heads (NIL32 << 32 | 0)
__global__ void __launch_bounds__(LC_T) lc_packprev_kernel(u64* prv, u64 n) {
  for (u64 v = (u64)blockIdx.x * LC_T + threadIdx.x; v < n; v += (u64)gridDim.x * LC_T) {
    const u64 u = prv[v];
    prv[v] = u == LC_NIL ? ((u64)LC_NIL32 << 32) : ((u << 32) | 1ull);
  }
}

// ranking waves, in place: v is final once its parent is (or it has none);
// the writer publishes dist[v] before the DONE mark (release), a child reads
// the mark (acquire) before the parent's dist, so finals may cascade inside
// a wave — the values are the same as the reference's snapshot waves.
__device__ __forceinline__ u64 ld_acquire_u64(const u64* p) {
  u64 v;
  asm volatile("ld.acquire.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_release_u64(u64* p, u64 v) {
  asm volatile("st.release.gpu.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}

__global__ void __launch_bounds__(LC_T) lc_wave_kernel(u64* nxt, u64* dist, u64 n, LcDev* d) {
  u32 pend = 0, fin = 0;
  for (u64 v = (u64)blockIdx.x * LC_T + threadIdx.x; v < n; v += (u64)gridDim.x * LC_T) {
    const u64 par = ld_acquire_u64(nxt + v);
    if (par == LC_DONE) continue;
    if (par == LC_NIL || ld_acquire_u64(nxt + par) == LC_DONE) {
      if (par != LC_NIL) dist[v] += dist[par];
      st_release_u64(nxt + v, LC_DONE);
      ++fin;
    } else {
      ++pend;
    }
  }
  pend = __reduce_add_sync(0xffffffffu, pend);
  fin = __reduce_add_sync(0xffffffffu, fin);
  if ((threadIdx.x & 31) == 0) {
    if (pend) atomicAdd((unsigned long long*)&d->pending, (unsigned long long)pend);
    if (fin) atomicAdd((unsigned long long*)&d->ready, (unsigned long long)fin);
  }
}

// ---------------------------------------------------------------------------
// tree contraction (contraction.py:368-525): the frontier queue and cursor
// (control plane, O(prefix) per round) stay on the host; these kernels do
// the per-node work of a round on the device-resident tree.

// contractible-when-swept flags for ids [lo, hi) (contraction.py:417-421)
__global__ void __launch_bounds__(LC_T) tc_ready_kernel(const u64* __restrict__ pa, const u64* __restrict__ lf,
                                                        const u64* __restrict__ rt, u64 lo, u64 hi,
                                                        unsigned char* flags) {
  for (u64 v = lo + (u64)blockIdx.x * LC_T + threadIdx.x; v < hi; v += (u64)gridDim.x * LC_T) {
    const bool l = lf[v] != LC_NIL, r = rt[v] != LC_NIL;
    const bool zero = !l && !r, unary = !l || !r;
    flags[v - lo] = (zero || (unary && pa[v] != LC_NIL)) ? 1 : 0;
  }
}

__device__ __forceinline__ bool tc_active(const u32* __restrict__ sorted, u64 fill, u64 x) {
  if (x == LC_NIL) return false;
  u64 lo = 0, hi = fill;
  while (lo < hi) {
    const u64 mid = (lo + hi) >> 1;
    if ((u64)sorted[mid] < x) lo = mid + 1;
    else hi = mid;
  }
  return lo < fill && (u64)sorted[lo] == x;
}

// eligibility (contraction.py:451-462)
__global__ void __launch_bounds__(LC_T) tc_elig_kernel(const u64* __restrict__ pa, const u64* __restrict__ lf,
                                                       const u64* __restrict__ rt, const u64* __restrict__ p,
                                                       const u32* __restrict__ ids, u64 fill,
                                                       const u32* __restrict__ sorted, unsigned char* elig) {
  for (u64 k = (u64)blockIdx.x * LC_T + threadIdx.x; k < fill; k += (u64)gridDim.x * LC_T) {
    const u64 v = ids[k];
    const u64 a = pa[v], l = lf[v], r = rt[v], pv = p[v];
    bool ok = (l == LC_NIL && r == LC_NIL) || a != LC_NIL;
    if (tc_active(sorted, fill, a)) ok = ok && pv < p[a];
    if (tc_active(sorted, fill, l)) ok = ok && pv < p[l];
    if (tc_active(sorted, fill, r)) ok = ok && pv < p[r];
    elig[k] = ok ? 1 : 0;
  }
}

// pre-surgery state of each committing node: parent, child, is_left, the
// parent's child count, the grandparent, the node's value
// (contraction.py:475-493)
static constexpr int TC_G = 6;  // gathered words per committing node

__global__ void __launch_bounds__(LC_T) tc_gather_kernel(const u64* __restrict__ pa, const u64* __restrict__ lf,
                                                         const u64* __restrict__ rt,
                                                         const u64* __restrict__ values,
                                                         const u32* __restrict__ vs, u64 nv, u64* out) {
  for (u64 k = (u64)blockIdx.x * LC_T + threadIdx.x; k < nv; k += (u64)gridDim.x * LC_T) {
    const u64 v = vs[k];
    const u64 a = pa[v], l = lf[v], r = rt[v];
    const u64 child = l != LC_NIL ? l : r;
    u64 is_left = 0, pre = 0, gp = LC_NIL;
    if (a != LC_NIL) {
      is_left = lf[a] == v;
      pre = (u64)(lf[a] != LC_NIL) + (u64)(rt[a] != LC_NIL);
      gp = pa[a];
    }
    out[TC_G * k] = a;
    out[TC_G * k + 1] = child;
    out[TC_G * k + 2] = is_left;
    out[TC_G * k + 3] = pre;
    out[TC_G * k + 4] = gp;
    out[TC_G * k + 5] = values[v];
  }
}

// value folding (rakes into the parent, compresses into the child) and the
// pointer surgery; writes are disjoint per committed node
__device__ __forceinline__ void tc_combine(u64* t, u64 x, int op) {
  unsigned long long* q = (unsigned long long*)t;
  if (op == 0) atomicAdd(q, (unsigned long long)x);
  else if (op == 1) atomicMax(q, (unsigned long long)x);
  else if (op == 2) atomicMin(q, (unsigned long long)x);
  else atomicXor(q, (unsigned long long)x);
}

__global__ void __launch_bounds__(LC_T) tc_commit_kernel(u64* pa, u64* lf, u64* rt, u64* values,
                                                         const u32* __restrict__ vs, u64 nv,
                                                         const u64* __restrict__ g, int op) {
  for (u64 k = (u64)blockIdx.x * LC_T + threadIdx.x; k < nv; k += (u64)gridDim.x * LC_T) {
    const u64 v = vs[k];
    const u64 a = g[TC_G * k], child = g[TC_G * k + 1], is_left = g[TC_G * k + 2];
    const u64 val = g[TC_G * k + 5];
    if (child != LC_NIL) tc_combine(values + child, val, op);
    else if (a != LC_NIL) tc_combine(values + a, val, op);
    if (a != LC_NIL) {
      if (is_left) lf[a] = child;
      else rt[a] = child;
    }
    if (child != LC_NIL) pa[child] = a;
  }
}

int tree_round_device(int step, u64* pa, u64* lf, u64* rt, const u64* p, u64* values, u64 lo, u64 hi,
                      const u32* ids, u64 fill, const u32* sorted, unsigned char* flags, u64* gathered,
                      int op, cudaStream_t st) {
  const int sms = num_sms(current_device());
  auto grid_for = [&](u64 items) {
    u64 g = (items + LC_T - 1) / LC_T;
    const u64 cap = (u64)sms * 8;
    return (unsigned)(g < 1 ? 1 : (g > cap ? cap : g));
  };
  switch (step) {
    case 0:  // ready flags of [lo, hi)
      if (hi > lo) tc_ready_kernel<<<grid_for(hi - lo), LC_T, 0, st>>>(pa, lf, rt, lo, hi, flags);
      break;
    case 1:  // eligibility of ids[0:fill)
      if (fill) tc_elig_kernel<<<grid_for(fill), LC_T, 0, st>>>(pa, lf, rt, p, ids, fill, sorted, flags);
      break;
    case 2:  // gather for the committing ids[0:fill)
      if (fill) tc_gather_kernel<<<grid_for(fill), LC_T, 0, st>>>(pa, lf, rt, values, ids, fill, gathered);
      break;
    case 3:  // fold + surgery
      if (fill) tc_commit_kernel<<<grid_for(fill), LC_T, 0, st>>>(pa, lf, rt, values, ids, fill, gathered, op);
      break;
    default:
      return PIP_ERR_INVALID_ARG;
  }
  PIP_CHECK_LAUNCH();
  return PIP_OK;
}

// ---------------------------------------------------------------------------
// host

struct LcLayout {
  size_t ids0, ids1, cflag, bcnt, dev, total;
};

static LcLayout lc_layout(u64 n, u64 prefix, bool rank) {
  LcLayout L{};
  size_t off = 0;
  auto take = [&](size_t bytes) {
    size_t o = off;
    off += (bytes + 255) & ~(size_t)255;
    return o;
  };
  const u64 P = prefix < n ? prefix : n;
  L.ids0 = take(P * 4);
  L.ids1 = take(P * 4);
  L.cflag = take(P);
  L.bcnt = take(((P + LC_BLK - 1) / LC_BLK) * 4);
  L.dev = take(sizeof(LcDev));
  L.total = off;
  return L;
}

size_t list_contract_workspace_bytes(u64 n, u64 prefix, int rank) {
  if (n == 0) return 0;
  if (prefix < 1) prefix = 1;
  return lc_layout(n, prefix, rank != 0).total;
}

// run the rounds; committed_per_round_host[r] for r < rounds_cap; trace_host
// (optional, host u64[n]) receives the committed ids round by round in packed
// order; splice_host (optional, host u64[3n]) receives (v, u, x) of each
// plain splice (on_splice); rank != 0: weighted variant + rank distribution
// (prv must hold the packed (prev << 32 | weight) form on entry).
int list_contract_device(u64* nxt, u64* prv, const u64* p, u64 n, u64 prefix, int rank,
                         u64* committed_per_round_host, u64 rounds_cap, u64* rounds_out,
                         u64* trace_host, u64* splice_host, void* ws, size_t ws_bytes, cudaStream_t st) {
  if (rounds_out) *rounds_out = 0;
  if (n == 0) return PIP_OK;
  if (n >= 0xffffffffull) return PIP_ERR_UNSUPPORTED;
  if (prefix < 1) return PIP_ERR_INVALID_ARG;
  const u64 P = prefix < n ? prefix : n;
  const LcLayout L = lc_layout(n, prefix, rank != 0);
  if (!ws || ws_bytes < L.total) return PIP_ERR_OOM;
  char* w = (char*)ws;
  u32* ids[2] = {(u32*)(w + L.ids0), (u32*)(w + L.ids1)};
  unsigned char* cflag = (unsigned char*)(w + L.cflag);
  u32* bcnt = (u32*)(w + L.bcnt);
  LcDev* d = (LcDev*)(w + L.dev);
  const int sms = num_sms(current_device());
  auto grid_for = [&](u64 items) {
    u64 g = (items + LC_T - 1) / LC_T;
    const u64 cap = (u64)sms * 8;
    return (unsigned)(g < 1 ? 1 : (g > cap ? cap : g));
  };
  if (rank) {
    lc_packprev_kernel<<<grid_for(n), LC_T, 0, st>>>(prv, n);
    PIP_CHECK_LAUNCH();
  }
  u64 cursor = 0, fill = 0, nfail = 0, rounds = 0, zero_rounds = 0, traced = 0;
  int cur = 0;
  std::vector<u32> hbuf;
  for (;;) {
    const u64 take = (P - nfail) < (n - cursor) ? (P - nfail) : (n - cursor);
    fill = nfail + take;
    if (fill == 0) break;
    const u64 c0 = cursor, c1 = cursor + take;
    PIP_CUDA(cudaMemsetAsync(&d->ncommit, 0, 8, st));
    if (rank) {
      lc_elig_kernel<true><<<grid_for(fill), LC_T, 0, st>>>(nxt, prv, p, ids[cur], cflag, fill, nfail, c0, c1);
      PIP_CHECK_LAUNCH();
      lc_splice_kernel<true><<<grid_for(fill), LC_T, 0, st>>>(nxt, prv, ids[cur], cflag, fill, d);
    } else {
      lc_elig_kernel<false><<<grid_for(fill), LC_T, 0, st>>>(nxt, prv, p, ids[cur], cflag, fill, nfail, c0, c1);
      PIP_CHECK_LAUNCH();
      lc_splice_kernel<false><<<grid_for(fill), LC_T, 0, st>>>(nxt, prv, ids[cur], cflag, fill, d);
    }
    PIP_CHECK_LAUNCH();
    u64 nc = 0;
    PIP_CUDA(cudaMemcpyAsync(&nc, &d->ncommit, 8, cudaMemcpyDeviceToHost, st));
    PIP_CUDA(cudaStreamSynchronize(st));
    cursor = c1;
    if (committed_per_round_host && rounds < rounds_cap) committed_per_round_host[rounds] = nc;
    if ((trace_host || splice_host) && nc) {
      // committed ids of this round, packed order (host bookkeeping for
      // trace / on_splice only)
      hbuf.resize(fill);
      std::vector<unsigned char> hf(fill);
      PIP_CUDA(cudaMemcpyAsync(hbuf.data(), ids[cur], fill * 4, cudaMemcpyDeviceToHost, st));
      PIP_CUDA(cudaMemcpyAsync(hf.data(), cflag, fill, cudaMemcpyDeviceToHost, st));
      PIP_CUDA(cudaStreamSynchronize(st));
      for (u64 k = 0; k < fill; ++k) {
        if (!hf[k]) continue;
        const u64 v = hbuf[k];
        if (trace_host) trace_host[traced] = v;
        if (splice_host) {
          u64 ux[2];
          PIP_CUDA(cudaMemcpy(&ux[0], prv + v, 8, cudaMemcpyDeviceToHost));
          PIP_CUDA(cudaMemcpy(&ux[1], nxt + v, 8, cudaMemcpyDeviceToHost));
          splice_host[3 * traced] = v;
          splice_host[3 * traced + 1] = ux[0];
          splice_host[3 * traced + 2] = ux[1];
        }
        ++traced;
      }
    }
    ++rounds;
    if (nc == 0) {
      if (++zero_rounds >= 64) {
        if (rounds_out) *rounds_out = rounds;
        return PIP_ERR_LIVELOCK;
      }
      nfail = fill;  // nothing retired: the prefix is unchanged
      continue;
    }
    zero_rounds = 0;
    nfail = fill - nc;
    if (nfail) {
      const u64 nblk = (fill + LC_BLK - 1) / LC_BLK;
      lc_count_kernel<<<(unsigned)nblk, LC_T, 0, st>>>(cflag, fill, bcnt);
      PIP_CHECK_LAUNCH();
      lc_scan_kernel<<<1, 1024, 0, st>>>(bcnt, nblk);
      PIP_CHECK_LAUNCH();
      lc_pack_kernel<<<(unsigned)nblk, LC_T, 0, st>>>(ids[cur], cflag, fill, bcnt, ids[cur ^ 1]);
      PIP_CHECK_LAUNCH();
      cur ^= 1;
    }
  }
  if (rounds_out) *rounds_out = rounds;
  if (!rank) return PIP_OK;
  // rank distribution: nxt = parent (or NIL), prv = distance to it
  for (u64 wave = 0;; ++wave) {
    PIP_CUDA(cudaMemsetAsync(&d->pending, 0, 16, st));
    lc_wave_kernel<<<grid_for(n), LC_T, 0, st>>>(nxt, prv, n, d);
    PIP_CHECK_LAUNCH();
    u64 hv[2];
    PIP_CUDA(cudaMemcpyAsync(hv, &d->pending, 16, cudaMemcpyDeviceToHost, st));
    PIP_CUDA(cudaStreamSynchronize(st));
    if (hv[0] == 0) break;
    if (hv[1] == 0) return PIP_ERR_INVALID_ARG;  // a dependence cycle (malformed list)
  }
  return PIP_OK;
}

}  // namespace pip
