// Multi-GPU entry points on an NCCL communicator (SURVEY.md §8(b) last
// bullet, §8(e)): the sharded scan and the sharded stable filter, one process
// per GPU, each rank owning one contiguous shard of the global array.
//
// The reference has no distributed code; the plans are the ones
// paper_2103_01216_b200/distributed.py runs over torch.distributed
// (sharded_scan / sharded_filter), restated over the NCCL C API so that any
// host language can drive them:
//   scan    local fold -> ncclAllGather of the shard totals (8 B per rank) ->
//           a one-thread kernel folds the totals of the lower ranks into the
//           carry -> in-place scan with a DEVICE carry-in.  Stream-ordered, no
//           host synchronization.
//   filter  local stable in-place filter -> ncclAllGather of the kept counts
//           -> (one host read of `world` counts: NCCL needs the message sizes)
//           -> the head of my kept words that belongs to lower shards leaves
//           by ncclSend straight out of the array -> the rest shifts down in
//           place (one pass) -> the words of higher ranks arrive by ncclRecv
//           straight into their final slots.  Destination precedes source at
//           rank granularity (strong.py:317-327's batching rule), every wait
//           points to a lower rank, so the chain resolves from rank 0 upwards.
// NCCL is resolved at run time (dlopen of the process's libnccl.so.2): the
// library has no link-time dependency on it and the single-GPU entry points
// work without it.
#include <dlfcn.h>
#include <cstdlib>
#include <vector>
#include "common.cuh"

namespace pip {

int scan_device(u64* a, u64 n, int op, u64 init, int inclusive, const u64* carry_dev,
                u64* total_dev, void* scratch, size_t scratch_bytes, cudaStream_t st);
int reduce_device(const u64* a, u64 n, int op, u64* total_dev, void* scratch, size_t scratch_bytes,
                  cudaStream_t st);
int filter_device(u64* a, u64 n, const pip_pred* pred, u64* m_dev, void* scratch,
                  size_t scratch_bytes, cudaStream_t st);
int move_device(u64* a, u64 dst, u64 src, u64 len, void* scratch, size_t scratch_bytes,
                cudaStream_t st);
int clear_stall(void* scratch, size_t scratch_bytes, cudaStream_t st);
int read_stall(const void* scratch, cudaStream_t st);

namespace {

// the slice of the NCCL API used here (nccl.h: ncclResult_t is an int enum,
// ncclSuccess = 0; ncclDataType_t ncclUint64 = 5)
struct NcclApi {
  int (*AllGather)(const void*, void*, size_t, int, void*, cudaStream_t) = nullptr;
  int (*Send)(const void*, size_t, int, int, void*, cudaStream_t) = nullptr;
  int (*Recv)(void*, size_t, int, int, void*, cudaStream_t) = nullptr;
  int (*GroupStart)() = nullptr;
  int (*GroupEnd)() = nullptr;
  int (*CommCount)(void*, int*) = nullptr;
  int (*CommUserRank)(void*, int*) = nullptr;
  bool ok = false;
};
constexpr int NCCL_U64 = 5;

const NcclApi& nccl() {
  static NcclApi api = [] {
    NcclApi a;
    void* h = nullptr;
    if (const char* e = getenv("PIP_NCCL_LIB")) h = dlopen(e, RTLD_NOW | RTLD_GLOBAL);
    // the copy the process already uses (torch's bundled one), else the system's
    if (!h) h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_NOLOAD);
    if (!h) h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
    if (!h) return a;
    a.AllGather = (decltype(a.AllGather))dlsym(h, "ncclAllGather");
    a.Send = (decltype(a.Send))dlsym(h, "ncclSend");
    a.Recv = (decltype(a.Recv))dlsym(h, "ncclRecv");
    a.GroupStart = (decltype(a.GroupStart))dlsym(h, "ncclGroupStart");
    a.GroupEnd = (decltype(a.GroupEnd))dlsym(h, "ncclGroupEnd");
    a.CommCount = (decltype(a.CommCount))dlsym(h, "ncclCommCount");
    a.CommUserRank = (decltype(a.CommUserRank))dlsym(h, "ncclCommUserRank");
    a.ok = a.AllGather && a.Send && a.Recv && a.GroupStart && a.GroupEnd && a.CommCount &&
           a.CommUserRank;
    return a;
  }();
  return api;
}

#define PIP_NCCL(call)                        \
  do {                                        \
    if ((call) != 0) return PIP_ERR_CUDA;     \
  } while (0)

// comm must be a communicator of `world` ranks in which this process is `rank`
int check_comm(const NcclApi& N, void* comm, int rank, int world) {
  if (!comm || world < 1 || rank < 0 || rank >= world) return PIP_ERR_INVALID_ARG;
  int c = 0, r = -1;
  PIP_NCCL(N.CommCount(comm, &c));
  PIP_NCCL(N.CommUserRank(comm, &r));
  return (c == world && r == rank) ? PIP_OK : PIP_ERR_INVALID_ARG;
}

__host__ __device__ inline u64 op_identity(int op) { return op == PIP_OP_MIN ? ~0ull : 0ull; }
__host__ __device__ inline u64 op_apply(int op, u64 x, u64 y) {
  switch (op) {
    case PIP_OP_ADD: return x + y;
    case PIP_OP_MAX: return x > y ? x : y;
    case PIP_OP_MIN: return x < y ? x : y;
    default: return x ^ y;
  }
}

__global__ void set_word_kernel(u64* p, u64 v) { *p = v; }

// totals[0:world) -> carry = fold of the lower ranks' totals, total = fold of all
__global__ void shard_carry_kernel(const u64* totals, int rank, int world, int op, u64* carry,
                                   u64* total) {
  u64 c = op_identity(op), t = op_identity(op);
  for (int r = 0; r < world; ++r) {
    if (r == rank) c = t;
    t = op_apply(op, t, totals[r]);
  }
  *carry = c;
  if (total) *total = t;
}

}  // namespace

// Movement plan of the sharded filter for `rank` (distributed.py filter_plan):
// counts[r] kept words in shard r = global [r*S, min(n,(r+1)*S)), S =
// ceil(n/world); rank's kept words local[0:c) go to global [O, O+c), O = the
// kept words of the lower ranks.
//   down: pieces of local[0:x) that land in lower shards (peer, local source
//         offset, length); stay: local[x:c) moves to local 0;
//   up:   pieces higher ranks send (peer, local destination offset, length).
int filter_shard_plan(const u64* counts, int world, int rank, u64 n_global,
                      std::vector<pip_shard_piece>& down, u64& stay_src, u64& stay_len,
                      std::vector<pip_shard_piece>& up) {
  if (!counts || world < 1 || rank < 0 || rank >= world) return PIP_ERR_INVALID_ARG;
  const u64 S = (n_global + (u64)world - 1) / (u64)world;
  auto lo_of = [&](int r) { const u64 v = (u64)r * S; return v < n_global ? v : n_global; };
  auto hi_of = [&](int r) { const u64 v = lo_of(r) + S; return v < n_global ? v : n_global; };
  std::vector<u64> offs((size_t)world + 1, 0);
  for (int r = 0; r < world; ++r) {
    if (counts[r] > hi_of(r) - lo_of(r)) return PIP_ERR_INVALID_ARG;
    offs[r + 1] = offs[r] + counts[r];
  }
  const u64 lo = lo_of(rank), hi = hi_of(rank), o = offs[rank], c = counts[rank];
  const u64 below = lo > o ? lo - o : 0;
  const u64 x = c < below ? c : below;  // my kept words landing below my shard
  down.clear();
  up.clear();
  for (int e = 0; e < rank; ++e) {
    const u64 g0 = o > lo_of(e) ? o : lo_of(e), g1 = (o + x) < hi_of(e) ? (o + x) : hi_of(e);
    if (g1 > g0) down.push_back({(uint32_t)e, 0u, g0 - o, g1 - g0});
  }
  stay_src = x;
  stay_len = c - x;
  for (int s = rank + 1; s < world; ++s) {
    const u64 g0 = offs[s] > lo ? offs[s] : lo, g1 = offs[s + 1] < hi ? offs[s + 1] : hi;
    if (g1 > g0) up.push_back({(uint32_t)s, 0u, g0 - lo, g1 - g0});
  }
  return PIP_OK;
}

}  // namespace pip

using namespace pip;

extern "C" {

size_t pip_sharded_workspace_bytes(int world) { return world < 1 ? 0 : 8 * ((size_t)world + 2); }

int pip_nccl_available(void) { return nccl().ok ? 1 : 0; }

int pip_scan_u64_sharded(uint64_t* a_local, uint64_t n_local, int op, uint64_t init, int inclusive,
                         void* nccl_comm, int rank, int world, void* workspace,
                         size_t workspace_bytes, uint64_t* total_dev, void* scratch,
                         size_t scratch_bytes, void* stream) {
  cudaStream_t st = (cudaStream_t)stream;
  if (op < PIP_OP_ADD || op > PIP_OP_XOR || (n_local && !a_local)) return PIP_ERR_INVALID_ARG;
  const NcclApi& N = nccl();
  if (!N.ok) return PIP_ERR_UNSUPPORTED;
  if (int rc = check_comm(N, nccl_comm, rank, world)) return rc;
  if (!workspace || workspace_bytes < pip_sharded_workspace_bytes(world)) return PIP_ERR_OOM;
  u64* totals = (u64*)workspace;  // [world] gathered, [world] mine / my carry
  u64* mine = totals + world;
  if (int rc = clear_stall(scratch, scratch_bytes, st)) return rc;
  if (n_local) {
    if (int rc = reduce_device((const u64*)a_local, n_local, op, mine, scratch, scratch_bytes, st))
      return rc;
  } else {
    set_word_kernel<<<1, 1, 0, st>>>(mine, op_identity(op));
    PIP_CHECK_LAUNCH();
  }
  PIP_NCCL(N.AllGather(mine, totals, 1, NCCL_U64, nccl_comm, st));
  shard_carry_kernel<<<1, 1, 0, st>>>(totals, rank, world, op, mine, (u64*)total_dev);
  PIP_CHECK_LAUNCH();
  if (!n_local) return PIP_OK;
  return scan_device((u64*)a_local, n_local, op, init, inclusive, mine, nullptr, scratch,
                     scratch_bytes, st);
}

int pip_filter_shard_plan(const uint64_t* counts, int world, int rank, uint64_t n_global,
                          pip_shard_piece* down, int* n_down, uint64_t* stay_src,
                          uint64_t* stay_len, pip_shard_piece* up, int* n_up) {
  if (!n_down || !n_up || !stay_src || !stay_len || (world > 1 && (!down || !up)))
    return PIP_ERR_INVALID_ARG;
  std::vector<pip_shard_piece> d, u;
  u64 ss = 0, sl = 0;
  if (int rc = filter_shard_plan((const u64*)counts, world, rank, n_global, d, ss, sl, u)) return rc;
  for (size_t k = 0; k < d.size(); ++k) down[k] = d[k];
  for (size_t k = 0; k < u.size(); ++k) up[k] = u[k];
  *n_down = (int)d.size();
  *n_up = (int)u.size();
  *stay_src = ss;
  *stay_len = sl;
  return PIP_OK;
}

int pip_filter_u64_sharded(uint64_t* a_local, uint64_t n_local, uint64_t n_global,
                           const pip_pred* pred, void* nccl_comm, int rank, int world,
                           void* workspace, size_t workspace_bytes, uint64_t* m_out,
                           uint64_t* local_len_out, void* scratch, size_t scratch_bytes,
                           void* stream) {
  cudaStream_t st = (cudaStream_t)stream;
  if (n_local && !a_local) return PIP_ERR_INVALID_ARG;
  const NcclApi& N = nccl();
  if (!N.ok) return PIP_ERR_UNSUPPORTED;
  if (int rc = check_comm(N, nccl_comm, rank, world)) return rc;
  if (!workspace || workspace_bytes < pip_sharded_workspace_bytes(world)) return PIP_ERR_OOM;
  {  // my shard must be the one the even split gives this rank
    const u64 S = (n_global + (u64)world - 1) / (u64)world;
    const u64 lo = (u64)rank * S < n_global ? (u64)rank * S : n_global;
    const u64 hi = lo + S < n_global ? lo + S : n_global;
    if (n_local != hi - lo) return PIP_ERR_INVALID_ARG;
  }
  u64* counts_dev = (u64*)workspace;
  u64* mine = counts_dev + world;
  if (int rc = clear_stall(scratch, scratch_bytes, st)) return rc;
  if (int rc = filter_device((u64*)a_local, n_local, pred, mine, scratch, scratch_bytes, st))
    return rc;
  PIP_NCCL(N.AllGather(mine, counts_dev, 1, NCCL_U64, nccl_comm, st));
  std::vector<u64> counts((size_t)world);
  PIP_CUDA(cudaMemcpyAsync(counts.data(), counts_dev, 8 * (size_t)world, cudaMemcpyDeviceToHost, st));
  PIP_CUDA(cudaStreamSynchronize(st));
  std::vector<pip_shard_piece> down, up;
  u64 ss = 0, sl = 0;
  if (int rc = filter_shard_plan(counts.data(), world, rank, n_global, down, ss, sl, up)) return rc;
  // 1. the head of my kept words goes to lower shards, straight from the array
  if (!down.empty()) {
    PIP_NCCL(N.GroupStart());
    int bad = 0;  // a failed call must not leave the group open
    for (const pip_shard_piece& p : down)
      bad |= N.Send(a_local + p.local_offset, p.length, NCCL_U64, (int)p.peer, nccl_comm, st);
    bad |= N.GroupEnd();
    if (bad) return PIP_ERR_CUDA;
  }
  // 2. what stays moves down to local 0 (one in-place pass)
  if (sl && ss)
    if (int rc = move_device((u64*)a_local, 0, ss, sl, scratch, scratch_bytes, st)) return rc;
  // 3. higher ranks' words land above what I kept, in their final slots
  if (!up.empty()) {
    PIP_NCCL(N.GroupStart());
    int bad = 0;
    for (const pip_shard_piece& p : up)
      bad |= N.Recv(a_local + p.local_offset, p.length, NCCL_U64, (int)p.peer, nccl_comm, st);
    bad |= N.GroupEnd();
    if (bad) return PIP_ERR_CUDA;
  }
  u64 m = 0;
  for (int r = 0; r < world; ++r) m += counts[r];
  if (m_out) *m_out = m;
  if (local_len_out) {  // words of the packed global prefix [0, m) that sit in my shard
    const u64 S = (n_global + (u64)world - 1) / (u64)world;
    const u64 lo = (u64)rank * S < n_global ? (u64)rank * S : n_global;
    *local_len_out = m > lo ? ((m - lo) < n_local ? (m - lo) : n_local) : 0;
  }
  return read_stall(scratch, st);
}

}  // extern "C"
