// extern "C" boundary (include/pip.h) and the host-buffer entry points.
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <mutex>
#include <vector>
#include "common.cuh"

namespace pip {

static thread_local char g_cuda_err[256] = "";
void set_cuda_error(cudaError_t e) {
  snprintf(g_cuda_err, sizeof(g_cuda_err), "%s: %s", cudaGetErrorName(e), cudaGetErrorString(e));
}

bool timing_enabled() {
  static int v = -1;
  if (v < 0) {
    const char* e = getenv("PIP_TIMING");
    v = (e && e[0] == '1') ? 1 : 0;
  }
  return v == 1;
}

// memory stride of the look-back slots: the scratch holds 4 slots per
// possible CTA (8 per SM); a grid of G CTAs uses 4G of them, so they can sit
// up to (8 x SMs) / G slots apart (PIP_LB_STRIDE overrides, for measurement)
u32 lb_stride(int sms, int grid) {
  u32 cap = grid > 0 ? (u32)((8 * sms) / grid) : 1u;
  if (cap < 1) cap = 1;
  u32 want = 4;  // measured: 4-8 apart saves ~7% of the scan at 2^32 over adjacent slots
  if (const char* e = getenv("PIP_LB_STRIDE")) want = (u32)atoi(e);
  if (want < 1) want = 1;
  return want < cap ? want : cap;
}

int current_device() {
  int d = 0;
  cudaGetDevice(&d);
  return d;
}

int num_sms(int device) {
  static int cache[64] = {0};
  if (device < 0 || device >= 64) device = 0;
  if (!cache[device]) {
    int v = 0;
    cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, device);
    cache[device] = v > 0 ? v : 1;
  }
  return cache[device];
}

size_t scratch_bytes_for(int sms);
int scan_device(u64* a, u64 n, int op, u64 init, int inclusive, const u64* carry_dev,
                u64* total_dev, void* scratch, size_t scratch_bytes, cudaStream_t st);
int reduce_device(const u64* a, u64 n, int op, u64* total_dev, void* scratch, size_t scratch_bytes,
                  cudaStream_t st);
int filter_device(u64* a, u64 n, const pip_pred* pred, u64* m_dev, void* scratch,
                  size_t scratch_bytes, cudaStream_t st);
int count_device(const u64* a, u64 n, const pip_pred* pred, u64* m_dev, void* scratch,
                 size_t scratch_bytes, cudaStream_t st);
int rotate_device(u64* a, u64 n, u64 o, cudaStream_t st);
int reverse_device(u64* a, u64 n, cudaStream_t st);
int move_device(u64* a, u64 dst, u64 src, u64 len, void* scratch, size_t scratch_bytes,
                cudaStream_t st);
int validate_device(const u64* h, u64 n, u64* nonself_dev, void* scratch, size_t scratch_bytes,
                    cudaStream_t st);
int rng_words(u64* out, u64 lo, u64 count, u64 seed, u32 shift, cudaStream_t st);
int make_swaps(u64* out, u64 lo, u64 count, u64 seed, cudaStream_t st);
int bench_random_rmw(u64* buf, u64 n, u64 updates, u64 seed, float* ms, cudaStream_t st, int mode);
size_t rp_workspace_bytes(u64 n, u64 prefix, int variant);
int rp_device(u64* a, const u64* h, u64 n, u64 prefix, int variant, int debug,
              u64* counts_host, u64 rounds_cap, u64* trace_dev, void* ws, size_t ws_bytes,
              pip_rp_stats* stats, cudaStream_t st, const RpProgress* prog = nullptr);
size_t partition_workspace_bytes(u64 n);
size_t list_contract_workspace_bytes(u64 n, u64 prefix, int rank);
size_t tree_contract_workspace_bytes(u64 n, u64 prefix);
int tree_contract_device(u64* pa, u64* lf, u64* rt, const u64* p, u64* values, u64 n, u64 prefix, int op,
                         int debug, u64* committed_per_round_host, u64 rounds_cap, u64* rounds_out,
                         u64* trace_host, u64* roots_host, u64* nroots_out, u64* violations_out, void* ws,
                         size_t ws_bytes, cudaStream_t st);
int tree_round_device(int step, u64* pa, u64* lf, u64* rt, const u64* p, u64* values, u64 lo, u64 hi,
                      const u32* ids, u64 fill, const u32* sorted, unsigned char* flags, u64* gathered,
                      int op, cudaStream_t st);
int list_contract_device(u64* nxt, u64* prv, const u64* p, u64 n, u64 prefix, int rank,
                         u64* committed_per_round_host, u64 rounds_cap, u64* rounds_out,
                         u64* trace_host, u64* splice_host, void* ws, size_t ws_bytes, cudaStream_t st);
int sort_segments_device(u64* a, const u64* seg_lo, const u32* seg_len, u64 nseg, cudaStream_t st);
int sort_segments_grid_device(u64* a, const u64* seg_lo, const u32* seg_len, u64 nseg,
                              u64 max_len, cudaStream_t st);
int partition_device(u64* a, u64 n, const pip_pred* pred, u64* m_dev, void* ws, size_t ws_bytes,
                     cudaStream_t st);
size_t merge_workspace_bytes(u64 n, u64 split, u64 budget_words);
int compact_mask_device(u64* a, u64 n, const unsigned char* mask, u64* m_dev, void* scratch,
                        size_t scratch_bytes, cudaStream_t st);
size_t rt_workspace_bytes(u64 n);
int rt_reserve_max(u64* tkeys, u64* tvals, u64 cap, const u64* keys, const u64* vals, u64 n,
                   void* ws, size_t ws_bytes, u64* count_out, cudaStream_t st);
int rt_lookup(const u64* tkeys, const u64* tvals, u64 cap, const u64* keys, u64 n, u64* out_vals,
              unsigned char* found, cudaStream_t st);
int rt_delete(u64* tkeys, u64 cap, const u64* keys, u64 n, void* ws, size_t ws_bytes, u64* count_out,
              cudaStream_t st);
int merge_copy_device(const u64* a, u64 na, const u64* b, u64 nb, u64* out, cudaStream_t st);
int merge_device(u64* a, u64 n, u64 split, int check_sorted, void* ws, size_t ws_bytes,
                 void* scratch, size_t scratch_bytes, cudaStream_t st);

// ---------------------------------------------------------------------------
// host-buffer helpers: device buffers come from a small per-device caching
// pool (the *_host entry points would otherwise pay cudaMalloc/cudaFree on
// every call, which dominates small inputs); RAII returns them to the pool.
struct PoolBlock {
  int dev;
  size_t bytes;
  void* p;
};
static std::mutex g_pool_mu;
static std::vector<PoolBlock> g_pool;
static const size_t POOL_KEEP = 16;

static cudaError_t pool_get(size_t bytes, void** out) {
  int dev = 0;
  cudaGetDevice(&dev);
  {
    std::lock_guard<std::mutex> lk(g_pool_mu);
    size_t best = (size_t)-1, bi = 0;
    for (size_t i = 0; i < g_pool.size(); ++i)
      if (g_pool[i].dev == dev && g_pool[i].bytes >= bytes && g_pool[i].bytes < best &&
          g_pool[i].bytes <= 4 * bytes + (1u << 20)) {
        best = g_pool[i].bytes;
        bi = i;
      }
    if (best != (size_t)-1) {
      *out = g_pool[bi].p;
      g_pool.erase(g_pool.begin() + bi);
      return cudaSuccess;
    }
  }
  return cudaMalloc(out, bytes);
}
static void pool_put(void* p, size_t bytes) {
  int dev = 0;
  cudaGetDevice(&dev);
  std::lock_guard<std::mutex> lk(g_pool_mu);
  g_pool.push_back({dev, bytes, p});
  while (g_pool.size() > POOL_KEEP) {  // drop the largest
    size_t bi = 0;
    for (size_t i = 1; i < g_pool.size(); ++i)
      if (g_pool[i].bytes > g_pool[bi].bytes) bi = i;
    cudaFree(g_pool[bi].p);
    g_pool.erase(g_pool.begin() + bi);
  }
}

struct DevBuf {
  void* p = nullptr;
  size_t bytes = 0;
  ~DevBuf() {
    if (p) pool_put(p, bytes);
  }
  cudaError_t alloc(size_t b) {
    bytes = b ? b : 16;
    return pool_get(bytes, &p);
  }
};
// A Stream drains its queued work before it is destroyed, so an early error
// return never hands a DevBuf back to the pool while a copy or kernel still
// uses it.  Every function declares its DevBufs BEFORE its Streams (locals
// are destroyed in reverse order: streams drain first, buffers return after).
struct Stream {
  cudaStream_t s = nullptr;
  ~Stream() {
    if (s) {
      cudaStreamSynchronize(s);
      cudaStreamDestroy(s);
    }
  }
  cudaError_t create() { return cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking); }
};
struct Event {
  cudaEvent_t e = nullptr;
  ~Event() {
    if (e) cudaEventDestroy(e);
  }
  cudaError_t create() { return cudaEventCreateWithFlags(&e, cudaEventDisableTiming); }
};

// The look-back ops' stall flag (scratch word 0).  It is cleared once per
// public call, never per launch: a scan's tail launch must not wipe a stall
// its main launch raised, nor a chunk of a host scan one of an earlier chunk.
// PIP_INJECT_STALL=1 raises it right after the clear (tests of the
// reporting path; the kernels then bail out of their first long wait).
int clear_stall(void* scratch, size_t scratch_bytes, cudaStream_t st) {
  if (!scratch || scratch_bytes < 64) return PIP_OK;  // the op reports OOM itself
  PIP_CUDA(cudaMemsetAsync(scratch, 0, 4, st));
  const char* e = getenv("PIP_INJECT_STALL");
  if (e && e[0] == '1') PIP_CUDA(cudaMemsetAsync(scratch, 1, 1, st));
  return PIP_OK;
}
int read_stall(const void* scratch, cudaStream_t st) {
  u32 h = 0;
  PIP_CUDA(cudaMemcpyAsync(&h, scratch, 4, cudaMemcpyDeviceToHost, st));
  PIP_CUDA(cudaStreamSynchronize(st));
  return h ? PIP_ERR_STALLED : PIP_OK;
}

// the device entry points' predicate checks, made before a host entry point
// queues any transfer (so an invalid predicate never leaves copies in flight)
static bool pred_ok(const pip_pred* p) {
  return p && p->kind <= PIP_PRED_EQ && !(p->kind == PIP_PRED_MOD_EQ && p->a == 0);
}

// words per pipeline stage of the host-buffer entry points (PIP_HOST_CHUNK_LOG2)
static u64 host_chunk() {
  static u64 c = 0;
  if (!c) {
    const char* e = getenv("PIP_HOST_CHUNK_LOG2");
    const int lg = e ? atoi(e) : 24;
    c = 1ull << (lg >= 16 && lg <= 30 ? lg : 24);  // invalid values: the default
  }
  return c;
}
static int host_nbuf() {
  const char* e = getenv("PIP_HOST_NBUF");
  const int v = e ? atoi(e) : 4;  // 2^24-word chunks x 4 buffers: best measured
  return v >= 2 && v <= 8 ? v : 4;
}

// scan over host memory: chunk k is copied in on `cp_in`, scanned on `comp`
// with the running carry (the previous chunk's inclusive fold) and copied
// out on `cp_out`; three chunk buffers keep all three engines busy.
int scan_host(u64* host, u64 n, int op, u64 init, int inclusive, u64* total_out, int device) {
  PIP_CUDA(cudaSetDevice(device));
  const int sms = num_sms(device);
  if (n == 0) {
    if (total_out) *total_out = init;
    return PIP_OK;
  }
  const u64 HOST_CHUNK = host_chunk();
  const u64 chunk = n < HOST_CHUNK ? n : HOST_CHUNK;
  const int nb = n > chunk ? host_nbuf() : 1;
  DevBuf bufs[8], scratch, carry;
  for (int i = 0; i < nb; ++i) PIP_CUDA(bufs[i].alloc(chunk * 8));
  const size_t sb = scratch_bytes_for(sms);
  PIP_CUDA(scratch.alloc(sb));
  PIP_CUDA(carry.alloc(16 * 8));
  Stream cin, comp, cout;
  PIP_CUDA(cin.create());
  PIP_CUDA(comp.create());
  PIP_CUDA(cout.create());
  const u64 nchunks = (n + chunk - 1) / chunk;
  std::vector<Event> in_done(nchunks), comp_done(nchunks), out_done(nchunks);
  u64* cr = (u64*)carry.p;  // cr[k & 1] = carry into chunk k
  if (int rc = clear_stall(scratch.p, sb, comp.s)) return rc;
  u64 ident = op == PIP_OP_MIN ? ~0ull : 0ull;
  PIP_CUDA(cudaMemcpyAsync(cr, &ident, 8, cudaMemcpyHostToDevice, comp.s));
  PIP_CUDA(cudaStreamSynchronize(comp.s));
  for (u64 k = 0; k < nchunks; ++k) {
    PIP_CUDA(in_done[k].create());
    PIP_CUDA(comp_done[k].create());
    PIP_CUDA(out_done[k].create());
    const u64 off = k * chunk, len = (n - off) < chunk ? (n - off) : chunk;
    u64* b = (u64*)bufs[k % nb].p;
    if (k >= (u64)nb) PIP_CUDA(cudaStreamWaitEvent(cin.s, out_done[k - nb].e, 0));
    PIP_CUDA(cudaMemcpyAsync(b, host + off, len * 8, cudaMemcpyHostToDevice, cin.s));
    PIP_CUDA(cudaEventRecord(in_done[k].e, cin.s));
    PIP_CUDA(cudaStreamWaitEvent(comp.s, in_done[k].e, 0));
    int rc = scan_device(b, len, op, init, inclusive, cr + (k & 1), cr + ((k + 1) & 1),
                         scratch.p, sb, comp.s);
    if (rc) return rc;
    PIP_CUDA(cudaEventRecord(comp_done[k].e, comp.s));
    PIP_CUDA(cudaStreamWaitEvent(cout.s, comp_done[k].e, 0));
    PIP_CUDA(cudaMemcpyAsync(host + off, b, len * 8, cudaMemcpyDeviceToHost, cout.s));
    PIP_CUDA(cudaEventRecord(out_done[k].e, cout.s));
  }
  u64 tot = 0;
  PIP_CUDA(cudaMemcpyAsync(&tot, cr + (nchunks & 1), 8, cudaMemcpyDeviceToHost, comp.s));
  PIP_CUDA(cudaStreamSynchronize(comp.s));
  PIP_CUDA(cudaStreamSynchronize(cout.s));
  if (int rc = read_stall(scratch.p, comp.s)) return rc;
  if (total_out) *total_out = tot;
  return PIP_OK;
}

// filter over host memory: chunk k is filtered on device; once its kept
// count is known the kept prefix goes back to host[m : m + kept), which lies
// inside the already-uploaded part of the array (m <= chunk start).
int filter_host(u64* host, u64 n, const pip_pred* pred, u64* m_out, int device) {
  PIP_CUDA(cudaSetDevice(device));
  const int sms = num_sms(device);
  if (n == 0) {
    if (m_out) *m_out = 0;
    return PIP_OK;
  }
  const u64 HOST_CHUNK = host_chunk();
  const u64 chunk = n < HOST_CHUNK ? n : HOST_CHUNK;
  const int nb = n > chunk ? host_nbuf() : 1;
  DevBuf bufs[8], scratch, counts;
  for (int i = 0; i < nb; ++i) PIP_CUDA(bufs[i].alloc(chunk * 8));
  const size_t sb = scratch_bytes_for(sms);
  PIP_CUDA(scratch.alloc(sb));
  const u64 nchunks = (n + chunk - 1) / chunk;
  PIP_CUDA(counts.alloc(nchunks * 8));
  u64* hc = nullptr;
  PIP_CUDA(cudaMallocHost(&hc, nchunks * 8));
  struct HostFree {
    u64* p;
    ~HostFree() { cudaFreeHost(p); }
  } hf{hc};
  Stream cin, comp, cout;
  PIP_CUDA(cin.create());
  PIP_CUDA(comp.create());
  PIP_CUDA(cout.create());
  std::vector<Event> in_done(nchunks), cnt_done(nchunks), out_done(nchunks);
  for (u64 k = 0; k < nchunks; ++k) {
    PIP_CUDA(in_done[k].create());
    PIP_CUDA(cnt_done[k].create());
    PIP_CUDA(out_done[k].create());
  }
  if (int rc = clear_stall(scratch.p, sb, comp.s)) return rc;
  u64 m = 0;
  auto issue = [&](u64 k) -> int {
    const u64 off = k * chunk, len = (n - off) < chunk ? (n - off) : chunk;
    u64* b = (u64*)bufs[k % nb].p;
    if (k >= (u64)nb) PIP_CUDA(cudaStreamWaitEvent(cin.s, out_done[k - nb].e, 0));
    PIP_CUDA(cudaMemcpyAsync(b, host + off, len * 8, cudaMemcpyHostToDevice, cin.s));
    PIP_CUDA(cudaEventRecord(in_done[k].e, cin.s));
    PIP_CUDA(cudaStreamWaitEvent(comp.s, in_done[k].e, 0));
    int rc = filter_device(b, len, pred, (u64*)counts.p + k, scratch.p, sb, comp.s);
    if (rc) return rc;
    PIP_CUDA(cudaMemcpyAsync(hc + k, (u64*)counts.p + k, 8, cudaMemcpyDeviceToHost, comp.s));
    PIP_CUDA(cudaEventRecord(cnt_done[k].e, comp.s));
    return PIP_OK;
  };
  const u64 ahead = (u64)nb - 1;
  for (u64 k = 0; k < nchunks && k <= ahead; ++k)
    if (int rc = issue(k)) return rc;
  for (u64 k = 0; k < nchunks; ++k) {
    PIP_CUDA(cudaEventSynchronize(cnt_done[k].e));
    const u64 kept = hc[k];
    u64* b = (u64*)bufs[k % nb].p;
    if (kept) PIP_CUDA(cudaMemcpyAsync(host + m, b, kept * 8, cudaMemcpyDeviceToHost, cout.s));
    PIP_CUDA(cudaEventRecord(out_done[k].e, cout.s));
    m += kept;
    if (k + 1 + ahead < nchunks)
      if (int rc = issue(k + 1 + ahead)) return rc;
  }
  PIP_CUDA(cudaStreamSynchronize(cout.s));
  if (int rc = read_stall(scratch.p, comp.s)) return rc;
  if (m_out) *m_out = m;
  return PIP_OK;
}

// merge over host memory, streamed: output chunk k (C words) is merged on the
// device from A[i_k, i_k+1) and B[j_k, j_k+1) into a ring buffer and copied
// back to host[kC, (k+1)C).  Uploads run in chunk order: before chunk k the
// device holds A up to min(na, (k+1)C) (every A word its host region will
// overwrite; A words only move right) and B up to j_k+1 (B words only move
// left, so that covers the B part of the region).  Every host word is read
// by an upload before the write-back that overwrites it: the write-back of
// chunk k waits for its merge, which waits for its uploads, and later
// uploads read only host[(k+1)C, n).  Co-ranks are taken on the host array
// before anything moves.
static u64 host_corank(const u64* a, u64 na, const u64* b, u64 nb, u64 r) {
  u64 lo = r > nb ? r - nb : 0, hi = r < na ? r : na;
  while (lo < hi) {
    const u64 mid = (lo + hi) >> 1;
    if (b[r - mid - 1] >= a[mid]) lo = mid + 1;
    else hi = mid;
  }
  return lo;
}

// the streamed merge's output ring: the only device memory besides the
// uploaded runs (the array's device copy is staging, like every *_host
// path's); kept within a relaxed budget (>= 2^16 words per buffer)
static u64 merge_host_chunk(u64 n, u64 budget_words, int nbuf) {
  u64 chunk = host_chunk();
  if (budget_words && chunk * (u64)nbuf > budget_words) {
    chunk = budget_words / (u64)nbuf;
    if (chunk < (1ull << 16)) chunk = 1ull << 16;
  }
  return chunk > n ? n : chunk;
}
static bool merge_host_inplace() {
  const char* e = getenv("PIP_MERGE_HOST_INPLACE");
  return e && atoi(e);
}
static u64 merge_host_ring_words(u64 n, u64 budget_words) {
  const int nbuf = host_nbuf();
  const u64 chunk = merge_host_chunk(n, budget_words, nbuf);
  const u64 nchunks = (n + chunk - 1) / chunk;
  const u64 nr = nchunks < (u64)nbuf ? nchunks : (u64)nbuf;
  return nr * chunk;
}
// a relaxed call whose budget the ring would exceed (small n: one chunk of
// n words; tiny budgets: the 2^16-word floor) merges in place on the device
// with the budgeted workspace instead
static bool merge_host_use_inplace(u64 n, u64 budget_words) {
  return merge_host_inplace() || (budget_words && merge_host_ring_words(n, budget_words) > budget_words);
}
size_t merge_host_workspace_bytes(u64 n, u64 split, u64 budget_words) {
  if (split > n || n < 2 || split == 0 || split == n) return 0;
  if (merge_host_use_inplace(n, budget_words)) return merge_workspace_bytes(n, split, budget_words);
  return (size_t)(merge_host_ring_words(n, budget_words) * 8);
}

int merge_host_stream(u64* host, u64 n, u64 split, u64 budget_words, int device) {
  const u64 na = split, nb = n - split;
  const int nbuf = host_nbuf();
  const u64 chunk = merge_host_chunk(n, budget_words, nbuf);
  const u64 nchunks = (n + chunk - 1) / chunk;
  std::vector<u64> ci(nchunks + 1);
  for (u64 k = 0; k <= nchunks; ++k) {
    const u64 r = k * chunk < n ? k * chunk : n;
    ci[k] = host_corank(host, na, host + na, nb, r);
  }
  DevBuf d, ring[8];
  PIP_CUDA(d.alloc(n * 8));
  const int nr = nchunks < (u64)nbuf ? (int)nchunks : nbuf;
  for (int i = 0; i < nr; ++i) PIP_CUDA(ring[i].alloc(chunk * 8));
  Stream cin, comp, cout;
  PIP_CUDA(cin.create());
  PIP_CUDA(comp.create());
  PIP_CUDA(cout.create());
  std::vector<Event> in_done(nchunks), comp_done(nchunks), out_done(nchunks);
  u64* dv = (u64*)d.p;
  u64 ua = 0, ub = 0;
  for (u64 k = 0; k < nchunks; ++k) {
    PIP_CUDA(in_done[k].create());
    PIP_CUDA(comp_done[k].create());
    PIP_CUDA(out_done[k].create());
    const u64 r0 = k * chunk, r1 = (k + 1) * chunk < n ? (k + 1) * chunk : n;
    const u64 i0 = ci[k], i1 = ci[k + 1], j0 = r0 - i0, j1 = r1 - i1;
    const u64 ta = r1 < na ? r1 : na;
    if (ta > ua) {
      PIP_CUDA(cudaMemcpyAsync(dv + ua, host + ua, (ta - ua) * 8, cudaMemcpyHostToDevice, cin.s));
      ua = ta;
    }
    if (j1 > ub) {
      PIP_CUDA(cudaMemcpyAsync(dv + na + ub, host + na + ub, (j1 - ub) * 8,
                               cudaMemcpyHostToDevice, cin.s));
      ub = j1;
    }
    PIP_CUDA(cudaEventRecord(in_done[k].e, cin.s));
    PIP_CUDA(cudaStreamWaitEvent(comp.s, in_done[k].e, 0));
    if (k >= (u64)nr) PIP_CUDA(cudaStreamWaitEvent(comp.s, out_done[k - nr].e, 0));
    u64* o = (u64*)ring[k % nr].p;
    if (int rc = merge_copy_device(dv + i0, i1 - i0, dv + na + j0, j1 - j0, o, comp.s)) return rc;
    PIP_CUDA(cudaEventRecord(comp_done[k].e, comp.s));
    PIP_CUDA(cudaStreamWaitEvent(cout.s, comp_done[k].e, 0));
    PIP_CUDA(cudaMemcpyAsync(host + r0, o, (r1 - r0) * 8, cudaMemcpyDeviceToHost, cout.s));
    PIP_CUDA(cudaEventRecord(out_done[k].e, cout.s));
  }
  PIP_CUDA(cudaStreamSynchronize(cout.s));
  return PIP_OK;
}

// unstable partition over host memory, streamed: chunks are uploaded from
// both ends of the array into a full device copy and partitioned there one
// by one (partition_device on the chunk); trues go back to host[0 : m) from
// the front, falses to host[m : n) from the back.  A word is written back
// only into a host range whose upload has completed (front chunks open
// [0, f), back chunks [bk, n)), so every host word is read before it is
// overwritten; the next chunk is taken from the side whose open room is
// smaller than the kept (resp. dropped) words expected to land there.
int partition_host_stream(u64* host, u64 n, const pip_pred* pred, u64* m_out, int device) {
  u64 chunk = host_chunk();
  if (chunk > n) chunk = n;
  const u64 nchunks = (n + chunk - 1) / chunk;
  DevBuf d, ws, cnt;
  PIP_CUDA(d.alloc(n * 8));
  const size_t wb = partition_workspace_bytes(chunk);
  PIP_CUDA(ws.alloc(wb));
  PIP_CUDA(cnt.alloc(nchunks * 8));
  u64* hc = nullptr;
  PIP_CUDA(cudaMallocHost(&hc, nchunks * 8));
  struct HostFree {
    u64* p;
    ~HostFree() { cudaFreeHost(p); }
  } hf{hc};
  Stream cin, comp, cout;
  PIP_CUDA(cin.create());
  PIP_CUDA(comp.create());
  PIP_CUDA(cout.create());
  std::vector<Event> in_done(nchunks), cnt_done(nchunks);
  std::vector<u64> off_of(nchunks), len_of(nchunks), gate_f(nchunks), gate_b(nchunks);
  u64* dv = (u64*)d.p;
  u64 fi = 0, bi = nchunks - 1, issued = 0;  // next front / back chunk index
  u64 f = 0, bk = n;                          // issued upload bounds
  u64 t_known = 0, f_known = 0, w_known = 0, w_flight = 0;
  auto issue = [&]() -> int {
    const double rho = w_known ? (double)t_known / (double)w_known : 0.5;
    const double t_est = (double)t_known + rho * (double)w_flight;
    const double f_est = (double)f_known + (1.0 - rho) * (double)w_flight;
    const bool front = (double)f - t_est <= (double)(n - bk) - f_est;
    const u64 j = front ? fi++ : bi--;
    const u64 off = j * chunk, len = (n - off) < chunk ? (n - off) : chunk;
    const u64 k = issued++;
    PIP_CUDA(in_done[k].create());
    PIP_CUDA(cnt_done[k].create());
    PIP_CUDA(cudaMemcpyAsync(dv + off, host + off, len * 8, cudaMemcpyHostToDevice, cin.s));
    PIP_CUDA(cudaEventRecord(in_done[k].e, cin.s));
    PIP_CUDA(cudaStreamWaitEvent(comp.s, in_done[k].e, 0));
    if (int rc = partition_device(dv + off, len, pred, (u64*)cnt.p + k, ws.p, wb, comp.s)) return rc;
    PIP_CUDA(cudaMemcpyAsync(hc + k, (u64*)cnt.p + k, 8, cudaMemcpyDeviceToHost, comp.s));
    PIP_CUDA(cudaEventRecord(cnt_done[k].e, comp.s));
    if (front) f = off + len;
    else bk = off;
    off_of[k] = off;
    len_of[k] = len;
    gate_f[k] = f == bk ? n : f;  // once both ends meet every word is open
    gate_b[k] = f == bk ? 0 : bk;
    w_flight += len;
    return PIP_OK;
  };
  struct Piece {
    u64 off, len;
  };
  std::vector<Piece> pt, pf;  // pending trues / falses, in production order
  size_t pt_head = 0, pf_head = 0;
  u64 wt = 0, wf = 0;  // words written back: trues from 0 up, falses from n down
  auto flush = [&](u64 gf, u64 gb) -> int {
    while (pt_head < pt.size() && wt < gf) {
      Piece& q = pt[pt_head];
      const u64 x = q.len < gf - wt ? q.len : gf - wt;
      PIP_CUDA(cudaMemcpyAsync(host + wt, dv + q.off, x * 8, cudaMemcpyDeviceToHost, cout.s));
      wt += x;
      q.off += x;
      q.len -= x;
      if (q.len == 0) ++pt_head;
    }
    while (pf_head < pf.size() && n - wf > gb) {
      Piece& q = pf[pf_head];
      const u64 room = n - wf - gb;
      const u64 x = q.len < room ? q.len : room;
      PIP_CUDA(cudaMemcpyAsync(host + (n - wf - x), dv + q.off + (q.len - x), x * 8,
                               cudaMemcpyDeviceToHost, cout.s));
      wf += x;
      q.len -= x;
      if (q.len == 0) ++pf_head;
    }
    return PIP_OK;
  };
  const u64 ahead = (u64)host_nbuf();
  while (issued < nchunks && issued < ahead)
    if (int rc = issue()) return rc;
  for (u64 k = 0; k < nchunks; ++k) {
    PIP_CUDA(cudaEventSynchronize(cnt_done[k].e));
    const u64 t = hc[k], len = len_of[k];
    t_known += t;
    f_known += len - t;
    w_known += len;
    w_flight -= len;
    if (t) pt.push_back(Piece{off_of[k], t});
    if (len - t) pf.push_back(Piece{off_of[k] + t, len - t});
    // chunk k's partition has finished, so every upload issued up to it has landed
    if (int rc = flush(gate_f[k], gate_b[k])) return rc;
    if (issued < nchunks)
      if (int rc = issue()) return rc;
  }
  if (wt != t_known || wf != f_known) return PIP_ERR_CUDA;  // every word placed
  PIP_CUDA(cudaStreamSynchronize(cout.s));
  *m_out = t_known;
  return PIP_OK;
}

}  // namespace pip

using namespace pip;

extern "C" {

int pip_version(void) { return 1; }

const char* pip_status_string(int s) {
  switch (s) {
    case PIP_OK: return "ok";
    case PIP_ERR_INVALID_ARG: return "invalid argument";
    case PIP_ERR_INVALID_SWAPS: return "invalid swap sequence: H[i] must lie in [0, i]";
    case PIP_ERR_LIVELOCK: return "no iterate committed for 64 rounds";
    case PIP_ERR_OOM: return "workspace or scratch too small";
    case PIP_ERR_CUDA: return "CUDA error";
    case PIP_ERR_UNSORTED: return "unsorted input run";
    case PIP_ERR_UNSUPPORTED: return "unsupported size or option";
    case PIP_ERR_TABLE: return "reservation table overfull; presize the table";
    case PIP_ERR_DEBUG_SWEEP: return "debug sweep: reservation slots not clean after a round";
    case PIP_ERR_STALLED: return "a CTA's bounded wait expired (look-back / dataflow stall); output incomplete";
    default: return "unknown status";
  }
}

const char* pip_last_cuda_error(void) { return g_cuda_err; }

size_t pip_scratch_bytes(int device) { return scratch_bytes_for(num_sms(device)); }

int pip_scratch_status(const void* scratch, void* stream) {
  if (!scratch) return PIP_ERR_INVALID_ARG;
  return read_stall(scratch, (cudaStream_t)stream);
}

int pip_scan_u64(uint64_t* a, uint64_t n, int op, uint64_t init, int inclusive, uint64_t* total_dev,
                 void* scratch, size_t scratch_bytes, void* stream) {
  if (int rc = clear_stall(scratch, scratch_bytes, (cudaStream_t)stream)) return rc;
  return scan_device((u64*)a, n, op, init, inclusive, nullptr, (u64*)total_dev, scratch,
                     scratch_bytes, (cudaStream_t)stream);
}

int pip_scan_u64_carry(uint64_t* a, uint64_t n, int op, uint64_t init, int inclusive,
                       const uint64_t* carry_dev, uint64_t* total_dev, void* scratch,
                       size_t scratch_bytes, void* stream) {
  if (int rc = clear_stall(scratch, scratch_bytes, (cudaStream_t)stream)) return rc;
  return scan_device((u64*)a, n, op, init, inclusive, (const u64*)carry_dev, (u64*)total_dev,
                     scratch, scratch_bytes, (cudaStream_t)stream);
}

int pip_reduce_u64(const uint64_t* a, uint64_t n, int op, uint64_t* total_dev, void* scratch,
                   size_t scratch_bytes, void* stream) {
  if (int rc = clear_stall(scratch, scratch_bytes, (cudaStream_t)stream)) return rc;
  return reduce_device((const u64*)a, n, op, (u64*)total_dev, scratch, scratch_bytes,
                       (cudaStream_t)stream);
}

int pip_scan_u64_host(uint64_t* host_a, uint64_t n, int op, uint64_t init, int inclusive,
                      uint64_t* total_out, int device) {
  if (op < PIP_OP_ADD || op > PIP_OP_XOR || (n && !host_a)) return PIP_ERR_INVALID_ARG;
  return scan_host((u64*)host_a, n, op, init, inclusive, (u64*)total_out, device);
}

int pip_filter_u64(uint64_t* a, uint64_t n, const pip_pred* pred, uint64_t* m_dev, void* scratch,
                   size_t scratch_bytes, void* stream) {
  if (int rc = clear_stall(scratch, scratch_bytes, (cudaStream_t)stream)) return rc;
  return filter_device((u64*)a, n, pred, (u64*)m_dev, scratch, scratch_bytes, (cudaStream_t)stream);
}

int pip_count_u64(const uint64_t* a, uint64_t n, const pip_pred* pred, uint64_t* m_dev,
                  void* scratch, size_t scratch_bytes, void* stream) {
  if (int rc = clear_stall(scratch, scratch_bytes, (cudaStream_t)stream)) return rc;
  return count_device((const u64*)a, n, pred, (u64*)m_dev, scratch, scratch_bytes,
                      (cudaStream_t)stream);
}

int pip_filter_u64_host(uint64_t* host_a, uint64_t n, const pip_pred* pred, uint64_t* m_out,
                        int device) {
  if (!pred_ok(pred) || (n && !host_a)) return PIP_ERR_INVALID_ARG;
  return filter_host((u64*)host_a, n, pred, (u64*)m_out, device);
}

int pip_compact_by_mask_u64(uint64_t* a, uint64_t n, const uint8_t* keep, uint64_t* m_dev,
                            void* scratch, size_t scratch_bytes, void* stream) {
  if (int rc = clear_stall(scratch, scratch_bytes, (cudaStream_t)stream)) return rc;
  return compact_mask_device((u64*)a, n, keep, (u64*)m_dev, scratch, scratch_bytes,
                             (cudaStream_t)stream);
}

size_t pip_rt_workspace_bytes(uint64_t n) { return rt_workspace_bytes(n); }

int pip_rt_reserve_max_u64(uint64_t* table_keys, uint64_t* table_vals, uint64_t capacity,
                           const uint64_t* keys, const uint64_t* vals, uint64_t n, void* workspace,
                           size_t workspace_bytes, uint64_t* count_out, void* stream) {
  return rt_reserve_max((u64*)table_keys, (u64*)table_vals, capacity, (const u64*)keys,
                        (const u64*)vals, n, workspace, workspace_bytes, (u64*)count_out,
                        (cudaStream_t)stream);
}

int pip_rt_lookup_u64(const uint64_t* table_keys, const uint64_t* table_vals, uint64_t capacity,
                      const uint64_t* keys, uint64_t n, uint64_t* vals_out, uint8_t* found_out,
                      void* stream) {
  return rt_lookup((const u64*)table_keys, (const u64*)table_vals, capacity, (const u64*)keys, n,
                   (u64*)vals_out, found_out, (cudaStream_t)stream);
}

int pip_rt_delete_u64(uint64_t* table_keys, uint64_t capacity, const uint64_t* keys, uint64_t n,
                      void* workspace, size_t workspace_bytes, uint64_t* count_out, void* stream) {
  return rt_delete((u64*)table_keys, capacity, (const u64*)keys, n, workspace, workspace_bytes,
                   (u64*)count_out, (cudaStream_t)stream);
}

int pip_reverse_u64(uint64_t* a, uint64_t n, void* stream) {
  if (n && !a) return PIP_ERR_INVALID_ARG;
  return reverse_device((u64*)a, n, (cudaStream_t)stream);
}

int pip_move_u64(uint64_t* a, uint64_t dst, uint64_t src, uint64_t len, void* scratch,
                 size_t scratch_bytes, void* stream) {
  if (int rc = clear_stall(scratch, scratch_bytes, (cudaStream_t)stream)) return rc;
  return move_device((u64*)a, dst, src, len, scratch, scratch_bytes, (cudaStream_t)stream);
}

int pip_rotate_u64(uint64_t* a, uint64_t n, uint64_t o, void* scratch, size_t scratch_bytes,
                   void* stream) {
  (void)scratch;
  (void)scratch_bytes;
  return rotate_device((u64*)a, n, o, (cudaStream_t)stream);
}

size_t pip_partition_workspace_bytes(uint64_t n) { return partition_workspace_bytes(n); }

int pip_tree_round_u64(int step, uint64_t* parent, uint64_t* left, uint64_t* right,
                       const uint64_t* p, uint64_t* values, uint64_t lo, uint64_t hi,
                       const uint32_t* ids, uint64_t fill, const uint32_t* sorted_ids,
                       uint8_t* flags, uint64_t* gathered, int combine, void* stream) {
  return tree_round_device(step, (u64*)parent, (u64*)left, (u64*)right, (const u64*)p, (u64*)values, lo,
                           hi, ids, fill, sorted_ids, flags, (u64*)gathered, combine,
                           (cudaStream_t)stream);
}

size_t pip_tree_contract_workspace_bytes(uint64_t n, uint64_t prefix) {
  return tree_contract_workspace_bytes(n, prefix);
}

int pip_tree_contract_u64(uint64_t* parent, uint64_t* left, uint64_t* right, const uint64_t* p,
                          uint64_t* values, uint64_t n, uint64_t prefix, int combine, int debug,
                          uint64_t* committed_per_round_host, uint64_t rounds_cap, uint64_t* rounds_out,
                          uint64_t* trace_host, uint64_t* roots_host, uint64_t* nroots_out,
                          uint64_t* violations_out, void* workspace, size_t workspace_bytes,
                          void* stream) {
  return tree_contract_device((u64*)parent, (u64*)left, (u64*)right, (const u64*)p, (u64*)values, n, prefix,
                              combine, debug, (u64*)committed_per_round_host, rounds_cap, (u64*)rounds_out,
                              (u64*)trace_host, (u64*)roots_host, (u64*)nroots_out, (u64*)violations_out,
                              workspace, workspace_bytes, (cudaStream_t)stream);
}

size_t pip_list_contract_workspace_bytes(uint64_t n, uint64_t prefix, int rank) {
  return list_contract_workspace_bytes(n, prefix, rank);
}

int pip_list_contract_u64(uint64_t* next, uint64_t* prev, const uint64_t* p, uint64_t n,
                          uint64_t prefix, int rank, uint64_t* committed_per_round_host,
                          uint64_t rounds_cap, uint64_t* rounds_out, uint64_t* trace_host,
                          uint64_t* splice_host, void* workspace, size_t workspace_bytes,
                          void* stream) {
  return list_contract_device((u64*)next, (u64*)prev, (const u64*)p, n, prefix, rank,
                              (u64*)committed_per_round_host, rounds_cap, (u64*)rounds_out,
                              (u64*)trace_host, (u64*)splice_host, workspace, workspace_bytes,
                              (cudaStream_t)stream);
}

int pip_sort_segments_u64(uint64_t* a, const uint64_t* seg_lo_dev, const uint32_t* seg_len_dev,
                          uint64_t nseg, void* stream) {
  return sort_segments_device((u64*)a, (const u64*)seg_lo_dev, seg_len_dev, nseg,
                              (cudaStream_t)stream);
}

int pip_sort_segments_grid_u64(uint64_t* a, const uint64_t* seg_lo_dev, const uint32_t* seg_len_dev,
                               uint64_t nseg, uint64_t max_len, void* stream) {
  return sort_segments_grid_device((u64*)a, (const u64*)seg_lo_dev, seg_len_dev, nseg, max_len,
                                   (cudaStream_t)stream);
}

int pip_partition_u64(uint64_t* a, uint64_t n, const pip_pred* pred, uint64_t* m_dev,
                      void* workspace, size_t workspace_bytes, void* stream) {
  return partition_device((u64*)a, n, pred, (u64*)m_dev, workspace, workspace_bytes,
                          (cudaStream_t)stream);
}

int pip_partition_segments_u64(uint64_t* a, const uint64_t* seg_lo, const uint64_t* seg_len,
                               const uint64_t* operand, uint32_t kind, uint64_t* m_dev,
                               uint64_t nseg, void* workspace, size_t workspace_bytes,
                               void* stream) {
  if (nseg && (!a || !seg_lo || !seg_len || !operand || !m_dev)) return PIP_ERR_INVALID_ARG;
  if (kind < PIP_PRED_LT || kind > PIP_PRED_EQ) return PIP_ERR_INVALID_ARG;
  for (uint64_t g = 0; g < nseg; ++g) {
    pip_pred p{kind, 0, operand[g], 0};
    const int rc = partition_device((u64*)a + seg_lo[g], seg_len[g], &p, (u64*)m_dev + g,
                                    workspace, workspace_bytes, (cudaStream_t)stream);
    if (rc) return rc;
  }
  return PIP_OK;
}

int pip_partition_u64_host(uint64_t* host_a, uint64_t n, const pip_pred* pred, uint64_t* m_out,
                           int device) {
  if (!pred_ok(pred) || !m_out || (n && !host_a)) return PIP_ERR_INVALID_ARG;
  PIP_CUDA(cudaSetDevice(device));
  if (n == 0) {
    *m_out = 0;
    return PIP_OK;
  }
  const char* e = getenv("PIP_PARTITION_HOST_INPLACE");
  if (!(e && atoi(e)) && n > host_chunk()) return partition_host_stream((u64*)host_a, n, pred, (u64*)m_out, device);
  DevBuf a, ws, m;
  Stream s;
  PIP_CUDA(s.create());
  PIP_CUDA(a.alloc(n * 8));
  const size_t wb = partition_workspace_bytes(n);
  PIP_CUDA(ws.alloc(wb));
  PIP_CUDA(m.alloc(8));
  PIP_CUDA(cudaMemcpyAsync(a.p, host_a, n * 8, cudaMemcpyHostToDevice, s.s));
  int rc = partition_device((u64*)a.p, n, pred, (u64*)m.p, ws.p, wb, s.s);
  if (rc) return rc;
  PIP_CUDA(cudaMemcpyAsync(host_a, a.p, n * 8, cudaMemcpyDeviceToHost, s.s));
  PIP_CUDA(cudaMemcpyAsync(m_out, m.p, 8, cudaMemcpyDeviceToHost, s.s));
  PIP_CUDA(cudaStreamSynchronize(s.s));
  return PIP_OK;
}

size_t pip_merge_workspace_bytes(uint64_t n, uint64_t split, uint64_t budget_words) {
  return merge_workspace_bytes(n, split, budget_words);
}

int pip_merge_u64(uint64_t* a, uint64_t n, uint64_t split, int check_sorted, void* workspace,
                  size_t workspace_bytes, void* scratch, size_t scratch_bytes, void* stream) {
  return merge_device((u64*)a, n, split, check_sorted, workspace, workspace_bytes, scratch,
                      scratch_bytes, (cudaStream_t)stream);
}

size_t pip_merge_host_workspace_bytes(uint64_t n, uint64_t split, uint64_t budget_words) {
  return merge_host_workspace_bytes(n, split, budget_words);
}

int pip_merge_u64_host(uint64_t* host_a, uint64_t n, uint64_t split, uint64_t budget_words,
                       int device) {
  if (split > n || (n && !host_a)) return PIP_ERR_INVALID_ARG;
  PIP_CUDA(cudaSetDevice(device));
  if (n < 2 || split == 0 || split == n) return PIP_OK;
  if (merge_host_use_inplace(n, budget_words)) {  // upload all, in-place device merge, copy back
    DevBuf a, ws, scratch;
    Stream s;
    PIP_CUDA(s.create());
    PIP_CUDA(a.alloc(n * 8));
    const size_t wb = merge_workspace_bytes(n, split, budget_words);
    PIP_CUDA(ws.alloc(wb));
    const size_t sb = scratch_bytes_for(num_sms(device));
    PIP_CUDA(scratch.alloc(sb));
    PIP_CUDA(cudaMemcpyAsync(a.p, host_a, n * 8, cudaMemcpyHostToDevice, s.s));
    int rc = merge_device((u64*)a.p, n, split, 0, wb ? ws.p : nullptr, wb, scratch.p, sb, s.s);
    if (rc) return rc;
    PIP_CUDA(cudaMemcpyAsync(host_a, a.p, n * 8, cudaMemcpyDeviceToHost, s.s));
    PIP_CUDA(cudaStreamSynchronize(s.s));
    return PIP_OK;
  }
  return merge_host_stream((u64*)host_a, n, split, budget_words, device);
}

size_t pip_rp_workspace_bytes(uint64_t n, uint64_t prefix, int variant) {
  return rp_workspace_bytes(n, prefix, variant);
}

int pip_random_permutation_u64(uint64_t* a, const uint64_t* h, uint64_t n, uint64_t prefix,
                               int variant, int debug, uint64_t* committed_per_round_host,
                               uint64_t rounds_cap, uint64_t* trace_dev, void* workspace,
                               size_t workspace_bytes, pip_rp_stats* stats_host, void* stream) {
  return rp_device((u64*)a, (const u64*)h, n, prefix, variant, debug,
                   (u64*)committed_per_round_host, rounds_cap, (u64*)trace_dev, workspace,
                   workspace_bytes, stats_host, (cudaStream_t)stream);
}

int pip_validate_swaps_u64(const uint64_t* h, uint64_t n, uint64_t* nonself_dev, void* scratch,
                           size_t scratch_bytes, void* stream) {
  return validate_device((const u64*)h, n, (u64*)nonself_dev, scratch, scratch_bytes,
                         (cudaStream_t)stream);
}

int pip_random_permutation_u64_host(uint64_t* host_a, const uint64_t* host_h, uint64_t n,
                                    uint64_t prefix, int variant, pip_rp_stats* stats_host,
                                    int device) {
  if (n && (!host_a || !host_h)) return PIP_ERR_INVALID_ARG;
  PIP_CUDA(cudaSetDevice(device));
  if (n == 0) {
    if (stats_host) memset(stats_host, 0, sizeof(*stats_host));
    return PIP_OK;
  }
  DevBuf a, h, ws;
  Stream s, cout;
  PIP_CUDA(s.create());
  PIP_CUDA(cout.create());
  PIP_CUDA(a.alloc(n * 8));
  PIP_CUDA(h.alloc(n * 8));
  const size_t wb = rp_workspace_bytes(n, prefix, variant);
  PIP_CUDA(ws.alloc(wb));
  PIP_CUDA(cudaMemcpyAsync(a.p, host_a, n * 8, cudaMemcpyHostToDevice, s.s));
  PIP_CUDA(cudaMemcpyAsync(h.p, host_h, n * 8, cudaMemcpyHostToDevice, s.s));
  // the final suffix a[top + 1 : n) goes back while the rounds run (in
  // pieces of >= 2^22 words; PIP_RP_HOST_OVERLAP=0 turns it off)
  const char* e = getenv("PIP_RP_HOST_OVERLAP");
  const bool overlap = !(e && atoi(e) == 0) && n >= (1ull << 23);
  struct Drain {
    u64* host;
    const u64* dev;
    cudaStream_t st;
    u64 lo;  // a[lo : n) has been queued
    cudaError_t err;
    static void hook(void* c, unsigned long long top) {
      Drain* d = (Drain*)c;
      const u64 from = top + 1;
      if (from < d->lo && d->lo - from >= (1ull << 22) && d->err == cudaSuccess) {
        d->err = cudaMemcpyAsync(d->host + from, d->dev + from, (d->lo - from) * 8,
                                 cudaMemcpyDeviceToHost, d->st);
        d->lo = from;
      }
    }
  } drain{(u64*)host_a, (const u64*)a.p, cout.s, n, cudaSuccess};
  unsigned long long* ph = nullptr;
  RpProgress prog{};
  if (overlap) {
    PIP_CUDA(cudaHostAlloc((void**)&ph, 8, cudaHostAllocMapped));
    *ph = n;
    unsigned long long* pd = nullptr;
    PIP_CUDA(cudaHostGetDevicePointer((void**)&pd, ph, 0));
    prog = RpProgress{pd, ph, &Drain::hook, &drain};
  }
  struct HostFree {
    unsigned long long* p;
    ~HostFree() {
      if (p) cudaFreeHost(p);
    }
  } hf{ph};
  int rc = rp_device((u64*)a.p, (const u64*)h.p, n, prefix, variant, 0, nullptr, 0, nullptr, ws.p,
                     wb, stats_host, s.s, overlap ? &prog : nullptr);
  if (rc) {
    // The drain already wrote final words of a[top+1 : n) back while the
    // host prefix still holds the input: bring the whole device state back
    // (the rounds run so far, a permutation of the input) so the caller's
    // array stays a permutation, as the reference's in-place swaps do.
    cudaStreamSynchronize(cout.s);
    if (cudaStreamSynchronize(s.s) == cudaSuccess &&
        cudaMemcpy(host_a, a.p, n * 8, cudaMemcpyDeviceToHost) != cudaSuccess)
      cudaGetLastError();
    return rc;
  }
  PIP_CUDA(drain.err);
  PIP_CUDA(cudaMemcpyAsync(host_a, a.p, drain.lo * 8, cudaMemcpyDeviceToHost, s.s));
  PIP_CUDA(cudaStreamSynchronize(s.s));
  PIP_CUDA(cudaStreamSynchronize(cout.s));
  return PIP_OK;
}

int pip_rng_words_u64(uint64_t* out, uint64_t lo, uint64_t count, uint64_t seed, uint32_t shift,
                      void* stream) {
  return rng_words((u64*)out, lo, count, seed, shift, (cudaStream_t)stream);
}

int pip_make_swaps_u64(uint64_t* out, uint64_t lo, uint64_t count, uint64_t seed, void* stream) {
  return make_swaps((u64*)out, lo, count, seed, (cudaStream_t)stream);
}

int pip_bench_random_rmw(uint64_t* buf, uint64_t n, uint64_t updates, uint64_t seed, float* ms_out,
                         void* stream) {
  return bench_random_rmw((u64*)buf, n, updates, seed, ms_out, (cudaStream_t)stream, -1);
}

int pip_bench_random_update(uint64_t* buf, uint64_t n, uint64_t updates, uint64_t seed, int form,
                            float* ms_out, void* stream) {
  if (form < 0 || form > 2) return PIP_ERR_INVALID_ARG;
  return bench_random_rmw((u64*)buf, n, updates, seed, ms_out, (cudaStream_t)stream, form);
}

}  // extern "C"
