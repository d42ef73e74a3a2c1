// Tree contraction with the whole round loop on the device
// (contraction.tree_contract, contraction.py:368-559, on detres.run_rounds,
// detres.py:256-307).
//
// The reference's client (_TreeClient) rakes leaves into their parents and
// compresses unary nodes into their child; its iterate source is a bounded
// frontier: a cursor sweeps the ids once in 4096-id blocks queueing nodes
// that are contractible when it passes (contraction.py:412-431), and a rake
// that leaves an already-swept parent contractible queues that parent
// (:539-545).  Every piece of that control plane lives in device memory
// here — the frontier ring, the active list (failures first, in order, then
// the ring's head), the active-id hash set of the eligibility test, the
// rake-parent map — and the host loop only reads a few counts per round:
//
//   sweep   ready counts per 4096-id block from the cursor; the host picks
//           how many blocks (and how many ids of the last one) fill the
//           frontier up to b(n) and where the cursor stops, exactly as the
//           reference's block loop; one kernel appends them in id order;
//   refill  the ring's head copied behind the failures (two D2D copies);
//   elig    active ids into a hash set; a node commits iff it is a bare
//           node or has a parent, and its priority is below every active
//           neighbour's (:450-462);
//   split   stable split of the list into committed ids (the round's trace
//           order) and failures (the next list);
//   gather  every committed node's pre-round state (parent, child, side,
//           the parent's child count and parent) before any surgery
//           (:475-493);
//   commit  value folding (atomic add / max / min / xor) and pointer
//           surgery; rakers count themselves into the rake-parent map;
//           bare nodes report (root, value) (:495-549);
//   pushes  the map's parents that became contractible and lie below the
//           cursor, sorted ascending (np.unique order), onto the ring.
//
// So rounds, committed-per-round, traces, roots, folded values and the final
// forest equal the reference's.
#include <cstdio>
#include <cstring>
#include <vector>
#include "common.cuh"

namespace pip {

static constexpr u64 TR_NIL = ~0ull;
static constexpr u32 TR_NIL32 = 0xffffffffu;
static constexpr int TR_T = 256;
static constexpr u64 TR_SWEEP = 4096;   // the reference's _SCAN_BLOCK
static constexpr u64 TR_PACK = 1024;    // items per split block
static constexpr u64 TR_MAXSB = 8192;   // sweep blocks per pass

int sort_segments_grid_device(u64* a, const u64* seg_lo, const u32* seg_len, u64 nseg, u64 max_len,
                              cudaStream_t st);

struct TrDev {
  u32 ncommit, npush, nroots, violations;
  u32 last_id, pad;
};

__device__ __forceinline__ u32 tr_home(u32 k, u32 logc) { return (u32)(((u64)k * GOLDEN) >> (64 - logc)); }

// insert (or find) key k; returns its slot
__device__ __forceinline__ u32 tr_insert(u32* keys, u32 logc, u32 k) {
  const u32 mask = (1u << logc) - 1u;
  u32 s = tr_home(k, logc);
  for (u32 step = 0; step <= mask; ++step) {
    const u32 prev = atomicCAS(keys + s, TR_NIL32, k);
    if (prev == TR_NIL32 || prev == k) return s;
    s = (s + 1) & mask;
  }
  return TR_NIL32;
}

__device__ __forceinline__ bool tr_member(const u32* keys, u32 logc, u64 k) {
  if (k == TR_NIL) return false;
  const u32 mask = (1u << logc) - 1u;
  u32 s = tr_home((u32)k, logc);
  for (u32 step = 0; step <= mask; ++step) {
    const u32 c = __ldcg(keys + s);
    if (c == (u32)k) return true;
    if (c == TR_NIL32) return false;
    s = (s + 1) & mask;
  }
  return false;
}

__device__ __forceinline__ bool tr_ready(const u64* pa, const u64* lf, const u64* rt, u64 v) {
  const bool l = lf[v] != TR_NIL, r = rt[v] != TR_NIL;
  // a root keeps collecting rakes until bare (contraction.py:417-421)
  return (!l && !r) || ((!l || !r) && pa[v] != TR_NIL);
}

__device__ __forceinline__ u32 tr_block_rank(bool f, u32* s_w, u32* tot) {
  const u32 lane = lane_id(), warp = warp_id();
  const u32 m = __ballot_sync(0xffffffffu, f);
  if (lane == 0) s_w[warp] = __popc(m);
  __syncthreads();
  if (warp == 0) {
    const u32 nw = TR_T / 32;
    const u32 v = lane < nw ? s_w[lane] : 0;
    u32 inc = v;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const u32 t = __shfl_up_sync(0xffffffffu, inc, o);
      if (lane >= (u32)o) inc += t;
    }
    if (lane < nw) s_w[lane] = inc - v;
    if (lane == 31) s_w[32] = inc;
  }
  __syncthreads();
  const u32 r = s_w[warp] + __popc(m & ((1u << lane) - 1u));
  *tot = s_w[32];
  __syncthreads();
  return r;
}

// ready counts of the sweep blocks [c0 + j*4096, ...) below c1
__global__ void __launch_bounds__(TR_T) tr_sweep_count(const u64* __restrict__ pa, const u64* __restrict__ lf,
                                                       const u64* __restrict__ rt, u64 c0, u64 c1, u32* cnt) {
  __shared__ u32 s_w[33];
  const u64 lo = c0 + (u64)blockIdx.x * TR_SWEEP;
  const u64 hi = lo + TR_SWEEP < c1 ? lo + TR_SWEEP : c1;
  u32 c = 0;
  for (u64 v = lo + threadIdx.x; v < hi; v += TR_T) c += tr_ready(pa, lf, rt, v);
  c = __reduce_add_sync(0xffffffffu, c);
  if (lane_id() == 0) s_w[warp_id()] = c;
  __syncthreads();
  if (threadIdx.x == 0) {
    u32 t = 0;
    for (int w = 0; w < TR_T / 32; ++w) t += s_w[w];
    cnt[blockIdx.x] = t;
  }
}

// append the ready ids of blocks 0..nb-1 (ascending; only `last_take` of
// the last block) to the ring at tail + off[j]; the last appended id goes
// to d->last_id
__global__ void __launch_bounds__(TR_T) tr_sweep_emit(const u64* __restrict__ pa, const u64* __restrict__ lf,
                                                      const u64* __restrict__ rt, u64 c0, u64 c1, u64 nb,
                                                      u32 last_take, const u32* __restrict__ off, u32* ring,
                                                      u64 Q, u64 tail, TrDev* d) {
  __shared__ u32 s_w[33];
  const u64 j = blockIdx.x;
  const u64 lo = c0 + j * TR_SWEEP;
  const u64 hi = lo + TR_SWEEP < c1 ? lo + TR_SWEEP : c1;
  const u32 cap = j + 1 == nb ? last_take : 0xffffffffu;
  u32 run = 0;
  for (u64 b0 = lo; b0 < hi; b0 += TR_T) {
    const u64 v = b0 + threadIdx.x;
    const bool f = v < hi && tr_ready(pa, lf, rt, v);
    u32 tot;
    const u32 r = run + tr_block_rank(f, s_w, &tot);
    if (f && r < cap) {
      ring[(tail + off[j] + r) % Q] = (u32)v;
      if (j + 1 == nb && r + 1 == cap) d->last_id = (u32)v;
    }
    run += tot;
  }
}

__global__ void tr_hash_ids(const u32* __restrict__ act, u64 fill, u32* keys, u32 logc) {
  for (u64 k = (u64)blockIdx.x * TR_T + threadIdx.x; k < fill; k += (u64)gridDim.x * TR_T)
    tr_insert(keys, logc, act[k]);
}

__global__ void tr_elig(const u64* __restrict__ pa, const u64* __restrict__ lf, const u64* __restrict__ rt,
                        const u64* __restrict__ p, const u32* __restrict__ act, u64 fill,
                        const u32* __restrict__ keys, u32 logc, unsigned char* cflag) {
  for (u64 k = (u64)blockIdx.x * TR_T + threadIdx.x; k < fill; k += (u64)gridDim.x * TR_T) {
    const u64 v = act[k];
    const u64 a = pa[v], l = lf[v], r = rt[v], pv = p[v];
    bool ok = (l == TR_NIL && r == TR_NIL) || a != TR_NIL;
    if (ok && tr_member(keys, logc, a)) ok = pv < p[a];
    if (ok && tr_member(keys, logc, l)) ok = pv < p[l];
    if (ok && tr_member(keys, logc, r)) ok = pv < p[r];
    cflag[k] = ok;
  }
}

// stable split: committed -> vs (order kept), failures -> nxt (order kept)
__global__ void __launch_bounds__(TR_T) tr_split_count(const unsigned char* __restrict__ cflag, u64 fill,
                                                       u32* bcnt) {
  __shared__ u32 s_w[33];
  const u64 lo = (u64)blockIdx.x * TR_PACK;
  u32 c = 0;
  for (u64 k = lo + threadIdx.x; k < lo + TR_PACK && k < fill; k += TR_T) c += cflag[k];
  c = __reduce_add_sync(0xffffffffu, c);
  if (lane_id() == 0) s_w[warp_id()] = c;
  __syncthreads();
  if (threadIdx.x == 0) {
    u32 t = 0;
    for (int w = 0; w < TR_T / 32; ++w) t += s_w[w];
    bcnt[blockIdx.x] = t;
  }
}

// exclusive scan of bcnt[0..nblk) by one CTA; total -> d->ncommit
__global__ void __launch_bounds__(1024) tr_split_scan(u32* bcnt, u64 nblk, TrDev* d) {
  __shared__ u32 s[1024];
  __shared__ u32 carry;
  if (threadIdx.x == 0) carry = 0;
  __syncthreads();
  for (u64 base = 0; base < nblk; base += 1024) {
    const u64 i = base + threadIdx.x;
    const u32 v = i < nblk ? bcnt[i] : 0;
    s[threadIdx.x] = v;
    __syncthreads();
    for (int o = 1; o < 1024; o <<= 1) {
      const u32 t = threadIdx.x >= (u32)o ? s[threadIdx.x - o] : 0;
      __syncthreads();
      s[threadIdx.x] += t;
      __syncthreads();
    }
    if (i < nblk) bcnt[i] = carry + s[threadIdx.x] - v;
    __syncthreads();
    if (threadIdx.x == 1023) carry += s[1023];
    __syncthreads();
  }
  if (threadIdx.x == 0) d->ncommit = carry;
}

// failures to nxt[0, nf) and the committed ids behind them, nxt[nf, fill)
// (the next round's refill overwrites those only after they are used)
__global__ void __launch_bounds__(TR_T) tr_split_scatter(const u32* __restrict__ act,
                                                         const unsigned char* __restrict__ cflag, u64 fill,
                                                         const u32* __restrict__ bcnt, u32* nxt,
                                                         const TrDev* __restrict__ d) {
  __shared__ u32 s_w[33];
  const u64 lo = (u64)blockIdx.x * TR_PACK;
  u32* vs = nxt + (fill - d->ncommit);
  u32 rc = bcnt[blockIdx.x];
  u32 rf = (u32)lo - rc;
  for (u64 b0 = lo; b0 < lo + TR_PACK && b0 < fill; b0 += TR_T) {
    const u64 k = b0 + threadIdx.x;
    const bool in = k < fill;
    const bool c = in && cflag[k];
    u32 tot;
    const u32 r = tr_block_rank(c, s_w, &tot);
    if (in) {
      if (c) vs[rc + r] = act[k];
      else nxt[rf + threadIdx.x - r] = act[k];  // failures before me in this chunk
    }
    rc += tot;
    rf += (u32)(fill - b0 < (u64)TR_T ? fill - b0 : (u64)TR_T) - tot;
  }
}

// pre-round state: w0 = parent32 | child32 << 32, w1 = grandparent32 |
// pre-child-count << 32 | is_left << 34.  (A committed node's own value is
// not folded into by any other commit of its round — its parent and child
// cannot commit with it — so the commit reads it directly.)
// the committed ids of the round sit at nxt[fill - ncommit, fill) (tr_split_scatter);
// their count is read on the device, so no host sync separates the split
// from the commits
__device__ __forceinline__ const u32* tr_committed(const u32* nxt, u64 fill, const TrDev* d, u64& nv) {
  nv = d->ncommit;
  return nxt + (fill - nv);
}

__global__ void tr_gather(const u64* __restrict__ pa, const u64* __restrict__ lf, const u64* __restrict__ rt,
                          const u32* __restrict__ nxt, u64 fill, const TrDev* __restrict__ d, u64* g) {
  u64 nv;
  const u32* vs = tr_committed(nxt, fill, d, nv);
  for (u64 k = (u64)blockIdx.x * TR_T + threadIdx.x; k < nv; k += (u64)gridDim.x * TR_T) {
    const u64 v = vs[k];
    const u64 a = pa[v], l = lf[v], r = rt[v];
    const u64 child = l != TR_NIL ? l : r;
    u64 is_left = 0, pre = 0, gp = TR_NIL;
    if (a != TR_NIL) {
      is_left = lf[a] == v;
      pre = (u64)(lf[a] != TR_NIL) + (u64)(rt[a] != TR_NIL);
      gp = pa[a];
    }
    g[2 * k] = (u64)(u32)a | ((u64)(u32)child << 32);
    g[2 * k + 1] = (u64)(u32)gp | (pre << 32) | (is_left << 34);
  }
}

__device__ __forceinline__ u64 tr_w(u32 x) { return x == TR_NIL32 ? TR_NIL : (u64)x; }

__device__ __forceinline__ void tr_combine(u64* t, u64 x, int op) {
  unsigned long long* q = (unsigned long long*)t;
  if (op == 0) atomicAdd(q, (unsigned long long)x);
  else if (op == 1) atomicMax(q, (unsigned long long)x);
  else if (op == 2) atomicMin(q, (unsigned long long)x);
  else atomicXor(q, (unsigned long long)x);
}

// debug sweep (contraction.py:481-485): committed ids into a set first
__global__ void tr_hash_committed(const u32* __restrict__ nxt, u64 fill, const TrDev* __restrict__ d,
                                  u32* keys, u32 logc) {
  u64 nv;
  const u32* vs = tr_committed(nxt, fill, d, nv);
  for (u64 k = (u64)blockIdx.x * TR_T + threadIdx.x; k < nv; k += (u64)gridDim.x * TR_T)
    tr_insert(keys, logc, vs[k]);
}

__global__ void tr_violations(const u32* __restrict__ nxt, u64 fill, const u64* __restrict__ g,
                              const u32* __restrict__ keys, u32 logc, TrDev* d) {
  u64 nv = d->ncommit;
  (void)nxt;
  (void)fill;
  u32 c = 0;
  for (u64 k = (u64)blockIdx.x * TR_T + threadIdx.x; k < nv; k += (u64)gridDim.x * TR_T)
    c += tr_member(keys, logc, tr_w((u32)g[2 * k]));
  c = __reduce_add_sync(0xffffffffu, c);
  if (lane_id() == 0 && c) atomicAdd(&d->violations, c);
}

// rake-parent map value: bits 0-7 rakes this round, 8-9 the parent's
// pre-round child count, 10 "the parent is a root"
__global__ void tr_commit(u64* pa, u64* lf, u64* rt, u64* values, const u32* __restrict__ nxt, u64 fill,
                          const u64* __restrict__ g, int op, u32* mkeys, u32* mval, u32 logm, u64* roots,
                          TrDev* d) {
  u64 nv;
  const u32* vs = tr_committed(nxt, fill, d, nv);
  for (u64 k = (u64)blockIdx.x * TR_T + threadIdx.x; k < nv; k += (u64)gridDim.x * TR_T) {
    const u64 v = vs[k];
    const u64 w0 = g[2 * k], w1 = g[2 * k + 1], val = values[v];
    const u64 a = tr_w((u32)w0), child = tr_w((u32)(w0 >> 32));
    const u64 gp = tr_w((u32)w1);
    const u32 pre = (u32)((w1 >> 32) & 3), is_left = (u32)((w1 >> 34) & 1);
    if (child != TR_NIL) tr_combine(values + child, val, op);
    else if (a != TR_NIL) tr_combine(values + a, val, op);
    if (a != TR_NIL) {
      if (is_left) lf[a] = child;
      else rt[a] = child;
    }
    if (child != TR_NIL) pa[child] = a;
    if (child == TR_NIL && a != TR_NIL) {  // a rake: count it into its parent
      const u32 s = tr_insert(mkeys, logm, (u32)a);
      if (s != TR_NIL32) {
        atomicOr(mval + s, (pre << 8) | ((gp == TR_NIL ? 1u : 0u) << 10));
        atomicAdd(mval + s, 1u);
      }
    }
    if (child == TR_NIL && a == TR_NIL) {  // bare: a finished root
      const u32 q = atomicAdd(&d->nroots, 1u);
      roots[2 * q] = v;
      roots[2 * q + 1] = val;
    }
  }
}

// the rake parents that became contractible below the cursor
__global__ void tr_collect(const u32* __restrict__ mkeys, const u32* __restrict__ mval, u64 cap, u64 cursor,
                           u64* list, TrDev* d) {
  for (u64 s = (u64)blockIdx.x * TR_T + threadIdx.x; s < cap; s += (u64)gridDim.x * TR_T) {
    const u32 key = mkeys[s];
    if (key == TR_NIL32) continue;
    const u32 mv = mval[s];
    const int pre = (int)((mv >> 8) & 3), post = pre - (int)(mv & 0xff);
    const bool want = ((mv >> 10) & 1) ? post == 0 : pre == 2;
    if (want && (u64)key < cursor) list[atomicAdd(&d->npush, 1u)] = key;
  }
}

__global__ void tr_push(const u64* __restrict__ list, u64 cnt, u32* ring, u64 Q, u64 tail) {
  for (u64 k = (u64)blockIdx.x * TR_T + threadIdx.x; k < cnt; k += (u64)gridDim.x * TR_T)
    ring[(tail + k) % Q] = (u32)list[k];
}

// ---------------------------------------------------------------------------
// host

struct TrLayout {
  size_t act0, act1, cflag, g, ring, scnt, soff, keys, vals, seg, bcnt, dev, total;
  u64 P, Q, hc, nsb;
  u32 logh;
};

// O(b(n)) device workspace, ~7 words per prefix slot: the two active lists
// (u32; the committed ids of a round sit behind the failures), flags, the
// gathered pre-round state (its space doubles as the push list), the
// frontier ring (the reference's 2 b + 8 entries, contraction.py:397), one
// hash table (>= 1.5 b slots) serving as the active-id set and then as the
// rake-parent map, sweep counts for <= 4 b ids per pass
static TrLayout tr_layout(u64 n, u64 prefix) {
  TrLayout L{};
  const u64 P = prefix < n ? prefix : n;
  L.P = P;
  L.Q = 2 * prefix + 8;
  L.logh = 3;
  while ((1ull << L.logh) < P + P / 2) ++L.logh;
  L.hc = 1ull << L.logh;
  L.nsb = (4 * P + TR_SWEEP - 1) / TR_SWEEP + 1;
  if (L.nsb > TR_MAXSB) L.nsb = TR_MAXSB;
  size_t off = 0;
  auto take = [&](size_t bytes) {
    size_t o = off;
    off += (bytes + 15) & ~(size_t)15;
    return o;
  };
  L.act0 = take(P * 4);
  L.act1 = take(P * 4);
  L.cflag = take(P);
  L.g = take(P * 16);
  L.ring = take(L.Q * 4);
  L.scnt = take(L.nsb * 4);
  L.soff = take(L.nsb * 4);
  L.keys = take(L.hc * 4);
  L.vals = take(L.hc * 4);
  L.seg = take(16);
  L.bcnt = take(((P + TR_PACK - 1) / TR_PACK) * 4);
  L.dev = take(sizeof(TrDev));
  L.total = off;
  return L;
}

size_t tree_contract_workspace_bytes(u64 n, u64 prefix) {
  if (n == 0) return 0;
  if (prefix < 1) prefix = 1;
  return tr_layout(n, prefix).total;
}

// roots_host: host u64[2 n] receiving (root, value) pairs, *nroots_out
// their count; trace_host (host u64[n], NULL ok): committed ids per round in
// packed order; *violations_out: debug count (debug != 0)
int tree_contract_device(u64* pa, u64* lf, u64* rt, const u64* p, u64* values, u64 n, u64 prefix, int op,
                         int debug, u64* committed_per_round_host, u64 rounds_cap, u64* rounds_out,
                         u64* trace_host, u64* roots_host, u64* nroots_out, u64* violations_out, void* ws,
                         size_t ws_bytes, cudaStream_t st) {
  if (rounds_out) *rounds_out = 0;
  if (nroots_out) *nroots_out = 0;
  if (violations_out) *violations_out = 0;
  if (n == 0) return PIP_OK;
  if (n >= 0xffffffffull) return PIP_ERR_UNSUPPORTED;
  if (prefix < 1 || op < 0 || op > 3 || !roots_host) return PIP_ERR_INVALID_ARG;
  const TrLayout L = tr_layout(n, prefix);
  if (!ws || ws_bytes < L.total) return PIP_ERR_OOM;
  char* w = (char*)ws;
  u32* act[2] = {(u32*)(w + L.act0), (u32*)(w + L.act1)};
  unsigned char* cflag = (unsigned char*)(w + L.cflag);
  u64* g = (u64*)(w + L.g);
  u64* list = g;  // the gathered state is dead once the commits ran
  u32* ring = (u32*)(w + L.ring);
  u32* scnt = (u32*)(w + L.scnt);
  u32* soff = (u32*)(w + L.soff);
  u32* hkeys = (u32*)(w + L.keys);
  u32* mval = (u32*)(w + L.vals);
  u64* seg = (u64*)(w + L.seg);
  u32* bcnt = (u32*)(w + L.bcnt);
  TrDev* d = (TrDev*)(w + L.dev);
  // finished roots go straight to page-locked host memory (transfer
  // staging, not device workspace)
  struct HostRoots {
    u64* h = nullptr;
    ~HostRoots() {
      if (h) cudaFreeHost(h);
    }
  } hr;
  PIP_CUDA(cudaHostAlloc((void**)&hr.h, L.P * 16 + 16, cudaHostAllocMapped));
  u64* roots = nullptr;
  PIP_CUDA(cudaHostGetDevicePointer((void**)&roots, hr.h, 0));
  const int sms = num_sms(current_device());
  auto grid_for = [&](u64 items) {
    u64 gg = (items + TR_T - 1) / TR_T;
    const u64 cap = (u64)sms * 8;
    return (unsigned)(gg < 1 ? 1 : (gg > cap ? cap : gg));
  };
  const u64 P = L.P, Q = L.Q;
  PIP_CUDA(cudaMemsetAsync(hkeys, 0xff, L.hc * 4, st));
  PIP_CUDA(cudaMemsetAsync(mval, 0, L.hc * 4, st));
  u64 qhead = 0, qsize = 0, cursor = 0;
  u64 nfail = 0, rounds = 0, zero_rounds = 0, traced = 0, nroots = 0, violations = 0;
  int cur = 0;
  std::vector<u32> hs(TR_MAXSB), ho(TR_MAXSB);
  TrDev hd{};
  for (;;) {
    // ---- the frontier sweep (contraction.py:412-431)
    while (qsize < P && cursor < n) {
      u64 need = P - qsize;
      u64 span = 4 * need;
      span = (span + TR_SWEEP - 1) / TR_SWEEP * TR_SWEEP;
      if (span < TR_SWEEP) span = TR_SWEEP;
      if (span > (L.nsb - 1) * TR_SWEEP) span = (L.nsb - 1) * TR_SWEEP;
      const u64 c1 = cursor + span < n ? cursor + span : n;
      const u64 nbk = (c1 - cursor + TR_SWEEP - 1) / TR_SWEEP;
      tr_sweep_count<<<(unsigned)nbk, TR_T, 0, st>>>(pa, lf, rt, cursor, c1, scnt);
      PIP_CHECK_LAUNCH();
      PIP_CUDA(cudaMemcpyAsync(hs.data(), scnt, nbk * 4, cudaMemcpyDeviceToHost, st));
      PIP_CUDA(cudaStreamSynchronize(st));
      u64 nb = 0, taken = 0, last_take = 0, new_cursor = c1;
      bool cut = false;
      for (u64 j = 0; j < nbk; ++j) {
        ho[j] = (u32)taken;
        const u64 c = hs[j];
        ++nb;
        if (c > need) {  // leave the surplus ahead of the cursor
          last_take = need;
          taken += need;
          cut = true;
          break;
        }
        taken += c;
        need -= c;
        last_take = c;
        new_cursor = cursor + (j + 1) * TR_SWEEP < n ? cursor + (j + 1) * TR_SWEEP : n;
        if (need == 0) break;
      }
      if (taken + qsize > Q) return PIP_ERR_TABLE;  // "frontier overflow" (contraction.py:405)
      if (taken) {
        PIP_CUDA(cudaMemcpyAsync(soff, ho.data(), nb * 4, cudaMemcpyHostToDevice, st));
        const u64 cend = cut ? c1 : new_cursor;
        tr_sweep_emit<<<(unsigned)nb, TR_T, 0, st>>>(pa, lf, rt, cursor, cend, nb, (u32)last_take, soff, ring, Q,
                                                     (qhead + qsize) % Q, d);
        PIP_CHECK_LAUNCH();
      }
      if (cut) {
        PIP_CUDA(cudaMemcpyAsync(&hd, d, sizeof(hd), cudaMemcpyDeviceToHost, st));
        PIP_CUDA(cudaStreamSynchronize(st));
        new_cursor = (u64)hd.last_id + 1;
      }
      qsize += taken;
      cursor = new_cursor;
    }
    // ---- refill: the ring's head behind the failures
    const u64 cnt = (P - nfail) < qsize ? (P - nfail) : qsize;
    if (cnt) {
      const u64 first = cnt < Q - qhead ? cnt : Q - qhead;
      PIP_CUDA(cudaMemcpyAsync(act[cur] + nfail, ring + qhead, first * 4, cudaMemcpyDeviceToDevice, st));
      if (first < cnt)
        PIP_CUDA(cudaMemcpyAsync(act[cur] + nfail + first, ring, (cnt - first) * 4, cudaMemcpyDeviceToDevice, st));
      qhead = (qhead + cnt) % Q;
      qsize -= cnt;
    }
    const u64 fill = nfail + cnt;
    if (fill == 0) break;
    // ---- eligibility
    tr_hash_ids<<<grid_for(fill), TR_T, 0, st>>>(act[cur], fill, hkeys, L.logh);
    tr_elig<<<grid_for(fill), TR_T, 0, st>>>(pa, lf, rt, p, act[cur], fill, hkeys, L.logh, cflag);
    PIP_CHECK_LAUNCH();
    PIP_CUDA(cudaMemsetAsync(hkeys, 0xff, L.hc * 4, st));
    // ---- split into committed (vs) and failures (next list)
    const u64 nblk = (fill + TR_PACK - 1) / TR_PACK;
    PIP_CUDA(cudaMemsetAsync(d, 0, sizeof(TrDev), st));
    tr_split_count<<<(unsigned)nblk, TR_T, 0, st>>>(cflag, fill, bcnt);
    tr_split_scan<<<1, 1024, 0, st>>>(bcnt, nblk, d);
    tr_split_scatter<<<(unsigned)nblk, TR_T, 0, st>>>(act[cur], cflag, fill, bcnt, act[cur ^ 1], d);
    PIP_CHECK_LAUNCH();
    // ---- gather, (debug) violations, fold + surgery, rake parents, roots:
    // sized for the whole list, each kernel reads the committed count itself
    const u32* nxt = act[cur ^ 1];
    tr_gather<<<grid_for(fill), TR_T, 0, st>>>(pa, lf, rt, nxt, fill, d, g);
    PIP_CHECK_LAUNCH();
    if (debug) {
      tr_hash_committed<<<grid_for(fill), TR_T, 0, st>>>(nxt, fill, d, hkeys, L.logh);
      tr_violations<<<grid_for(fill), TR_T, 0, st>>>(nxt, fill, g, hkeys, L.logh, d);
      PIP_CHECK_LAUNCH();
      PIP_CUDA(cudaMemsetAsync(hkeys, 0xff, L.hc * 4, st));
    }
    tr_commit<<<grid_for(fill), TR_T, 0, st>>>(pa, lf, rt, values, nxt, fill, g, op, hkeys, mval, L.logh, roots,
                                               d);
    PIP_CHECK_LAUNCH();
    tr_collect<<<grid_for(L.hc), TR_T, 0, st>>>(hkeys, mval, L.hc, cursor, list, d);
    PIP_CHECK_LAUNCH();
    // the round's one host sync: committed count, pushes, roots
    PIP_CUDA(cudaMemcpyAsync(&hd, d, sizeof(hd), cudaMemcpyDeviceToHost, st));
    PIP_CUDA(cudaStreamSynchronize(st));
    PIP_CUDA(cudaMemsetAsync(hkeys, 0xff, L.hc * 4, st));
    PIP_CUDA(cudaMemsetAsync(mval, 0, L.hc * 4, st));
    const u64 nv = hd.ncommit;
    if (committed_per_round_host && rounds < rounds_cap) committed_per_round_host[rounds] = nv;
    if (trace_host && nv) {
      std::vector<u32> t(nv);
      PIP_CUDA(cudaMemcpy(t.data(), nxt + (fill - nv), nv * 4, cudaMemcpyDeviceToHost));
      for (u64 k = 0; k < nv; ++k) trace_host[traced + k] = t[k];
    }
    traced += nv;
    ++rounds;
    violations += hd.violations;
    if (hd.nroots) {
      memcpy(roots_host + 2 * nroots, hr.h, (size_t)hd.nroots * 16);
      nroots += hd.nroots;
    }
    const u64 np = hd.npush;
    if (np) {
      if (qsize + np > Q) return PIP_ERR_TABLE;
      if (np > 1) {  // np.unique order: ascending ids
        const u64 sg[2] = {0, np};
        const u32 sl = (u32)np;
        PIP_CUDA(cudaMemcpyAsync(seg, &sg[0], 8, cudaMemcpyHostToDevice, st));
        PIP_CUDA(cudaMemcpyAsync((u32*)(seg + 1), &sl, 4, cudaMemcpyHostToDevice, st));
        if (int rc = sort_segments_grid_device(list, seg, (const u32*)(seg + 1), 1, np, st)) return rc;
      }
      tr_push<<<grid_for(np), TR_T, 0, st>>>(list, np, ring, Q, (qhead + qsize) % Q);
      PIP_CHECK_LAUNCH();
      qsize += np;
    }
    if (nv == 0) {
      if (++zero_rounds >= 64) {
        if (rounds_out) *rounds_out = rounds;
        return PIP_ERR_LIVELOCK;
      }
      nfail = fill;  // nothing retired: the list is unchanged
      continue;
    }
    zero_rounds = 0;
    nfail = fill - nv;
    cur ^= 1;
  }
  if (rounds_out) *rounds_out = rounds;
  if (nroots_out) *nroots_out = nroots;
  if (violations_out) *violations_out = violations;
  return PIP_OK;
}

}  // namespace pip
