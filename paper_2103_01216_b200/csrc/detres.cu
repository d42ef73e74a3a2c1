// Device write-max reservation table (detres.ReservationTable,
// /root/reference/pkg/src/pipal/detres.py:40-211).
//
// Layout: keys u64[cap], vals u64[cap] in device memory, cap a power of two,
// NIL = 2^64-1 marks an empty slot; home(k) = (k * GOLDEN) >> (64 - log2 cap)
// (detres.py:77-78), linear probing.
//
// reserve_max reproduces the reference's batch algorithm step for step, so
// the slot layout (which key sits in which slot) is the reference's, not
// just the key -> value map: in probe step s every pending key looks at its
// current slot; the slots that were EMPTY at the start of the step are
// claimed by the smallest contending key (write-min on the key word, NIL
// being the largest word, detres.py:117-124); every key that now finds
// itself in its slot takes the max of the slot's value and its own; the
// others move one slot on.  A step is four launches so that "empty at the
// start of the step" is a snapshot (kernel A), all claims land before the
// winners are known (B), a fresh slot's stale value is reset before the max
// (C: the reference assigns the value of a freshly claimed slot), and the
// max and the advance run last (D).  Duplicate keys in a batch follow the
// same probe path and meet in the same slot, so no dedupe pass is needed
// (the reference sorts to dedupe, :97-113).
#include "common.cuh"

namespace pip {

static constexpr u64 RT_NIL = ~0ull;
enum : unsigned char { RT_PENDING = 0, RT_PENDING_EMPTY = 1, RT_DONE = 2 };

__device__ __forceinline__ u64 rt_home(u64 k, u32 shift) { return (k * GOLDEN) >> shift; }

__global__ void rt_init_kernel(const u64* __restrict__ keys, u64 n, u32 shift, u64* slot,
                               unsigned char* state) {
  for (u64 i = blockIdx.x * (u64)blockDim.x + threadIdx.x; i < n; i += (u64)gridDim.x * blockDim.x) {
    slot[i] = rt_home(keys[i], shift);
    state[i] = RT_PENDING;
  }
}

// A: snapshot which pending keys look at an empty slot
__global__ void rt_snapshot_kernel(const u64* __restrict__ tkeys, u64 n, const u64* __restrict__ slot,
                                   unsigned char* state) {
  for (u64 i = blockIdx.x * (u64)blockDim.x + threadIdx.x; i < n; i += (u64)gridDim.x * blockDim.x)
    if (state[i] != RT_DONE) state[i] = tkeys[slot[i]] == RT_NIL ? RT_PENDING_EMPTY : RT_PENDING;
}

// B: claim the snapshot-empty slots by write-min on the key word
__global__ void rt_claim_kernel(u64* tkeys, const u64* __restrict__ keys, u64 n,
                                const u64* __restrict__ slot, const unsigned char* __restrict__ state) {
  for (u64 i = blockIdx.x * (u64)blockDim.x + threadIdx.x; i < n; i += (u64)gridDim.x * blockDim.x)
    if (state[i] == RT_PENDING_EMPTY) atomicMin(&tkeys[slot[i]], keys[i]);
}

// C: the winners of a fresh slot reset its (stale) value
__global__ void rt_fresh_kernel(const u64* __restrict__ tkeys, u64* tvals, const u64* __restrict__ keys,
                                u64 n, const u64* __restrict__ slot, const unsigned char* __restrict__ state) {
  for (u64 i = blockIdx.x * (u64)blockDim.x + threadIdx.x; i < n; i += (u64)gridDim.x * blockDim.x)
    if (state[i] == RT_PENDING_EMPTY && tkeys[slot[i]] == keys[i]) tvals[slot[i]] = 0;
}

// D: hits take the max; misses advance; count what is still pending
__global__ void rt_max_kernel(const u64* __restrict__ tkeys, u64* tvals, const u64* __restrict__ keys,
                              const u64* __restrict__ vals, u64 n, u64 mask, u64* slot,
                              unsigned char* state, u32* pending) {
  u32 mine = 0;
  for (u64 i = blockIdx.x * (u64)blockDim.x + threadIdx.x; i < n; i += (u64)gridDim.x * blockDim.x) {
    if (state[i] == RT_DONE) continue;
    const u64 s = slot[i];
    if (tkeys[s] == keys[i]) {
      atomicMax(&tvals[s], vals[i]);
      state[i] = RT_DONE;
    } else {
      slot[i] = (s + 1) & mask;
      state[i] = RT_PENDING;
      ++mine;
    }
  }
  mine = __reduce_add_sync(0xffffffffu, mine);
  if ((threadIdx.x & 31) == 0 && mine) atomicAdd(pending, mine);
}

__global__ void rt_count_kernel(const u64* __restrict__ tkeys, u64 cap, u64* out) {
  u64 mine = 0;
  for (u64 i = blockIdx.x * (u64)blockDim.x + threadIdx.x; i < cap; i += (u64)gridDim.x * blockDim.x)
    mine += tkeys[i] != RT_NIL;
  for (int o = 16; o; o >>= 1) mine += __shfl_down_sync(0xffffffffu, mine, o);
  if ((threadIdx.x & 31) == 0 && mine) atomicAdd(out, mine);
}

// probe for each key: value + found (lookup, detres.py:130-163), or the slot
// it sits in (delete's locate pass, :165-193: every slot is located before
// any is cleared, so probe chains stay intact)
__global__ void rt_probe_kernel(const u64* __restrict__ tkeys, const u64* __restrict__ tvals, u64 cap,
                                u32 shift, const u64* __restrict__ keys, u64 n, u64* out_vals,
                                unsigned char* found, u64* out_slot) {
  const u64 mask = cap - 1;
  for (u64 i = blockIdx.x * (u64)blockDim.x + threadIdx.x; i < n; i += (u64)gridDim.x * blockDim.x) {
    const u64 k = keys[i];
    u64 s = rt_home(k, shift), v = RT_NIL, at = RT_NIL;
    for (u64 step = 0; step <= cap; ++step) {
      const u64 c = tkeys[s];
      if (c == k) {
        v = tvals[s];
        at = s;
        break;
      }
      if (c == RT_NIL) break;
      s = (s + 1) & mask;
    }
    if (out_vals) out_vals[i] = v;
    if (found) found[i] = at != RT_NIL;
    if (out_slot) out_slot[i] = at;
  }
}

__global__ void rt_clear_slots_kernel(u64* tkeys, const u64* __restrict__ slots, u64 n) {
  for (u64 i = blockIdx.x * (u64)blockDim.x + threadIdx.x; i < n; i += (u64)gridDim.x * blockDim.x)
    if (slots[i] != RT_NIL) tkeys[slots[i]] = RT_NIL;
}

static int rt_grid(u64 n) {
  const u64 g = (n + 255) / 256;
  const u64 cap = (u64)num_sms(current_device()) * 8;
  return (int)(g < 1 ? 1 : (g > cap ? cap : g));
}

static bool rt_pow2(u64 cap) { return cap >= 8 && (cap & (cap - 1)) == 0; }
static u32 rt_shift(u64 cap) { return (u32)(64 - (63 - __builtin_clzll(cap))); }

static int rt_count(const u64* tkeys, u64 cap, u64* scratch_word, u64* count_out, cudaStream_t st) {
  PIP_CUDA(cudaMemsetAsync(scratch_word, 0, 8, st));
  rt_count_kernel<<<rt_grid(cap), 256, 0, st>>>(tkeys, cap, scratch_word);
  PIP_CHECK_LAUNCH();
  PIP_CUDA(cudaMemcpyAsync(count_out, scratch_word, 8, cudaMemcpyDeviceToHost, st));
  PIP_CUDA(cudaStreamSynchronize(st));
  return PIP_OK;
}

size_t rt_workspace_bytes(u64 n) { return 64 + n * 9 + 16; }

int rt_reserve_max(u64* tkeys, u64* tvals, u64 cap, const u64* keys, const u64* vals, u64 n,
                   void* ws, size_t ws_bytes, u64* count_out, cudaStream_t st) {
  if (!rt_pow2(cap) || !tkeys || !tvals || !count_out || (n && (!keys || !vals)))
    return PIP_ERR_INVALID_ARG;
  if (n == 0) return rt_count(tkeys, cap, (u64*)ws, count_out, st);
  if (!ws || ws_bytes < rt_workspace_bytes(n)) return PIP_ERR_OOM;
  u64* word = (u64*)ws;  // [0]: count scratch, [1]: pending counter
  u32* pending = (u32*)(word + 1);
  u64* slot = word + 8;
  unsigned char* state = (unsigned char*)(slot + n);
  const u32 shift = rt_shift(cap);
  const int g = rt_grid(n);
  rt_init_kernel<<<g, 256, 0, st>>>(keys, n, shift, slot, state);
  PIP_CHECK_LAUNCH();
  u32 left = 1;
  for (u64 step = 0; left; ++step) {
    if (step > cap) return PIP_ERR_TABLE;  // "probe overflow" (detres.py:126-127)
    rt_snapshot_kernel<<<g, 256, 0, st>>>(tkeys, n, slot, state);
    rt_claim_kernel<<<g, 256, 0, st>>>(tkeys, keys, n, slot, state);
    rt_fresh_kernel<<<g, 256, 0, st>>>(tkeys, tvals, keys, n, slot, state);
    PIP_CUDA(cudaMemsetAsync(pending, 0, 4, st));
    rt_max_kernel<<<g, 256, 0, st>>>(tkeys, tvals, keys, vals, n, cap - 1, slot, state, pending);
    PIP_CHECK_LAUNCH();
    PIP_CUDA(cudaMemcpyAsync(&left, pending, 4, cudaMemcpyDeviceToHost, st));
    PIP_CUDA(cudaStreamSynchronize(st));
  }
  return rt_count(tkeys, cap, word, count_out, st);
}

int rt_lookup(const u64* tkeys, const u64* tvals, u64 cap, const u64* keys, u64 n, u64* out_vals,
              unsigned char* found, cudaStream_t st) {
  if (!rt_pow2(cap) || !tkeys || !tvals || (n && (!keys || !out_vals || !found)))
    return PIP_ERR_INVALID_ARG;
  if (n == 0) return PIP_OK;
  rt_probe_kernel<<<rt_grid(n), 256, 0, st>>>(tkeys, tvals, cap, rt_shift(cap), keys, n, out_vals,
                                              found, nullptr);
  PIP_CHECK_LAUNCH();
  return PIP_OK;
}

int rt_delete(u64* tkeys, u64 cap, const u64* keys, u64 n, void* ws, size_t ws_bytes, u64* count_out,
              cudaStream_t st) {
  if (!rt_pow2(cap) || !tkeys || !count_out || (n && !keys)) return PIP_ERR_INVALID_ARG;
  if (!ws || ws_bytes < rt_workspace_bytes(n)) return PIP_ERR_OOM;
  u64* word = (u64*)ws;
  u64* slot = word + 8;
  if (n) {
    rt_probe_kernel<<<rt_grid(n), 256, 0, st>>>(tkeys, nullptr, cap, rt_shift(cap), keys, n, nullptr,
                                                nullptr, slot);
    rt_clear_slots_kernel<<<rt_grid(n), 256, 0, st>>>(tkeys, slot, n);
    PIP_CHECK_LAUNCH();
  }
  return rt_count(tkeys, cap, word, count_out, st);
}

}  // namespace pip
