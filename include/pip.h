/*
 * pip.h — C ABI of the B200-native parallel in-place (PIP) kernels.
 *
 * This is the drop-in boundary for the reference's hot path
 * (`pipal`, /root/reference/pkg/src/pipal).  The reference is pure Python on
 * numpy uint64 arrays; its "plugin API" is the module-level functions listed
 * next to each entry point below.  A Python host layer
 * (paper_2103_01216_b200/) binds these entry points through ctypes and keeps
 * the reference's signatures, argument meaning and error behaviour; any
 * other FFI (cgo, JNI, N-API) can bind the same symbols — see INTEGRATION.md.
 *
 * Conventions
 *   - every array is a plain pointer to 64-bit words plus an element count;
 *   - `*_u64` entry points take DEVICE pointers and are stream-ordered on the
 *     given cudaStream_t (passed as void*, NULL = legacy default stream);
 *     device results (totals, counts) are written to DEVICE pointers;
 *   - `*_host` entry points take HOST pointers, run synchronously on a device
 *     of the caller's choice and include the host<->device transfers
 *     (chunked and overlapped where the algorithm streams);
 *   - nothing allocates device memory except the `*_host` entry points:
 *     auxiliary space comes from caller-provided `scratch` (O(#CTAs) bytes,
 *     independent of n: the analogue of the reference's unmetered recursion
 *     stack) and `workspace` (sublinear, metered by the caller — the analogue
 *     of runtime.alloc / runtime.release);
 *   - values are unsigned 64-bit; comparisons are unsigned (the reference
 *     compares numpy uint64), sums wrap mod 2^64.
 *   - every function returns a pip_status.
 */
#ifndef PIP_H_
#define PIP_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

enum pip_status {
  PIP_OK = 0,
  PIP_ERR_INVALID_ARG = 1,   /* reference: ValueError (bad split/offset/...) */
  PIP_ERR_INVALID_SWAPS = 2, /* reference: ValueError, H[i] must lie in [0,i] */
  PIP_ERR_LIVELOCK = 3,      /* reference: detres.LivelockError */
  PIP_ERR_OOM = 4,           /* workspace / scratch too small */
  PIP_ERR_CUDA = 5,          /* CUDA runtime error (see pip_last_cuda_error) */
  PIP_ERR_UNSORTED = 6,      /* reference: ValueError("unsorted input run") */
  PIP_ERR_UNSUPPORTED = 7,   /* size or option outside this build's support */
  PIP_ERR_TABLE = 8,         /* reservation table overfull (never in practice) */
  PIP_ERR_DEBUG_SWEEP = 9,   /* reference: debug sweep assertion failed */
  PIP_ERR_STALLED = 10       /* a CTA's bounded spin expired (look-back / dataflow
                                wait): the output is incomplete; see
                                pip_scratch_status */
};

/* scan element operations (strong.scan `op`): None/add, max, min, xor */
enum pip_scan_op { PIP_OP_ADD = 0, PIP_OP_MAX = 1, PIP_OP_MIN = 2, PIP_OP_XOR = 3 };

/* random-permutation storage variants (relaxed.RP_VARIANTS) */
enum pip_rp_variant { PIP_RP_NAIVE = 0, PIP_RP_FLAT = 1, PIP_RP_ONERES = 2, PIP_RP_FINAL = 3 };

/* Predicate descriptor replacing the reference's numpy callables
 * (cli.py:41 EVEN, test_strong.py:21,184, strong.py:440-441,553).
 * keep(x) = negate XOR test(x), with
 *   PIP_PRED_MASK_EQ : (x & a) == b          (even: a=1,b=0; odd: a=1,b=1)
 *   PIP_PRED_MOD_EQ  : (x % a) == b          (a >= 1; u64 magic division)
 *   PIP_PRED_LT/LE/GT/GE/EQ : x op a         (unsigned)
 *   PIP_PRED_ALL     : true
 */
enum pip_pred_kind {
  PIP_PRED_ALL = 0, PIP_PRED_MASK_EQ = 1, PIP_PRED_MOD_EQ = 2, PIP_PRED_LT = 3,
  PIP_PRED_LE = 4, PIP_PRED_GT = 5, PIP_PRED_GE = 6, PIP_PRED_EQ = 7
};
typedef struct pip_pred {
  uint32_t kind;
  uint32_t negate;
  uint64_t a;
  uint64_t b;
} pip_pred;

/* Round statistics of the deterministic-reservations engine
 * (detres.RoundStats, detres.py:222-230). */
typedef struct pip_rp_stats {
  uint64_t rounds;             /* RoundStats.rounds */
  uint64_t total_committed;    /* RoundStats.total_committed */
  uint64_t n_iterates;         /* non-self swaps (relaxed.py:239) */
  uint64_t peak_table_count;   /* max distinct keys held by the table in a round */
  uint64_t table_capacity;     /* reference capacity: peak_table_load = count/capacity */
  uint64_t prefix;             /* b(n) used */
  uint64_t workspace_words;    /* device workspace the run used, in 64-bit words */
  uint64_t rounds_recorded;    /* committed-per-round entries written */
} pip_rp_stats;

/* ---- library / sizing ---------------------------------------------------- */
int pip_version(void);
const char* pip_status_string(int status);
const char* pip_last_cuda_error(void);
/* bytes of O(#CTAs) scratch every strong op needs on `device` */
size_t pip_scratch_bytes(int device);
/* Status of the stream-ordered look-back ops (pip_scan_u64*, pip_reduce_u64,
 * pip_filter_u64, pip_count_u64) that last ran on `scratch`: synchronizes
 * `stream` and returns PIP_ERR_STALLED when a CTA of one of them gave up
 * waiting (its spin bound expired; the output is then incomplete), else
 * PIP_OK.  Each of those entry points clears the flag when it is queued, so
 * call this after every call whose result is used (the Python layer does).
 * The *_host entry points and the merge / permutation check it themselves. */
int pip_scratch_status(const void* scratch, void* stream);

/* ---- scan: strong.scan / strong.scan_blocked (strong.py:151-236) --------- *
 * Exclusive (inclusive=0) or inclusive in-place scan of a[0:n) under `op`.
 * Exclusive output: a[i] = op(init, x0 op ... op x_{i-1}), a[0] = init
 * (reference: op=None -> init 0; op given -> init = `identity`).
 * Inclusive output: a[i] = op(init, x0 op ... op x_i).
 * total_dev (device, may be NULL) receives x0 op ... op x_{n-1} (no init).
 * Replaces strong.py:151-166 (scan) and :169-236 (scan_blocked).           */
int pip_scan_u64(uint64_t* a, uint64_t n, int op, uint64_t init, int inclusive,
                 uint64_t* total_dev, void* scratch, size_t scratch_bytes, void* stream);
/* Same, with a DEVICE carry-in: outputs are op(init, op(*carry_dev, ...))
 * and total_dev receives op(*carry_dev, x0 .. x_{n-1}) — the running carry a
 * sharded or chunked scan hands to the next shard/chunk without a host sync. */
int pip_scan_u64_carry(uint64_t* a, uint64_t n, int op, uint64_t init, int inclusive,
                       const uint64_t* carry_dev, uint64_t* total_dev, void* scratch,
                       size_t scratch_bytes, void* stream);
/* Fold without writing (strong.reduce, strong.py:43-64; shard totals). */
int pip_reduce_u64(const uint64_t* a, uint64_t n, int op, uint64_t* total_dev,
                   void* scratch, size_t scratch_bytes, void* stream);
/* Host-buffer scan: H2D / scan-with-carry / D2H pipelined in chunks. */
int pip_scan_u64_host(uint64_t* host_a, uint64_t n, int op, uint64_t init, int inclusive,
                      uint64_t* total_out, int device);

/* ---- filter: strong.filter_kway / relaxed.filter_relaxed ----------------- *
 * Stable in-place filter of a[0:n): kept values end in a[0:m) in original
 * order; a[m:n) is unspecified (as in the reference).  m_dev (device)
 * receives m.  Replaces strong.py:283-349 and relaxed.py:284-309.          */
int pip_filter_u64(uint64_t* a, uint64_t n, const pip_pred* pred, uint64_t* m_dev,
                   void* scratch, size_t scratch_bytes, void* stream);
/* Count kept elements without moving anything (shard counts). */
int pip_count_u64(const uint64_t* a, uint64_t n, const pip_pred* pred, uint64_t* m_dev,
                  void* scratch, size_t scratch_bytes, void* stream);
int pip_filter_u64_host(uint64_t* host_a, uint64_t n, const pip_pred* pred, uint64_t* m_out,
                        int device);

/* ---- runtime.compact_by_mask (runtime.py:335-355) ------------------------ *
 * Stable in-place compaction: a[0:m) = the a[i] with keep[i] != 0 (device
 * byte mask u8[n]), in order; m to device m_dev; a[m:n) unspecified.  The
 * failure packing of the round engine (detres.py:303).  Same look-back
 * scratch and status rules as pip_filter_u64.                               */
int pip_compact_by_mask_u64(uint64_t* a, uint64_t n, const uint8_t* keep, uint64_t* m_dev,
                            void* scratch, size_t scratch_bytes, void* stream);

/* ---- detres.ReservationTable (detres.py:40-211) on the device ------------- *
 * table_keys / table_vals: device u64[capacity], capacity a power of two
 * >= 8, empty slots hold NIL = 2^64-1 in table_keys; home(k) =
 * (k * 0x9E3779B97F4A7C15) >> (64 - log2 capacity), linear probing.
 * reserve_max: per key, slot value = max(existing, written values) — the
 * reference's batch algorithm step by step (claims of empty slots by
 * write-min on the key word), so the slot layout equals the reference's;
 * keys / vals device u64[n]; workspace holds pip_rt_workspace_bytes(n);
 * *count_out (HOST) receives the occupied slots afterwards; synchronizes;
 * PIP_ERR_TABLE on probe overflow (detres.py:126-127).
 * lookup: vals_out (device u64[n], NIL when absent) and found_out (device
 * u8[n]); stream-ordered.  delete: clears the keys' slots (all located
 * before any is cleared, :165-193); *count_out (HOST) as above.           */
size_t pip_rt_workspace_bytes(uint64_t n);
int pip_rt_reserve_max_u64(uint64_t* table_keys, uint64_t* table_vals, uint64_t capacity,
                           const uint64_t* keys, const uint64_t* vals, uint64_t n, void* workspace,
                           size_t workspace_bytes, uint64_t* count_out, void* stream);
int pip_rt_lookup_u64(const uint64_t* table_keys, const uint64_t* table_vals, uint64_t capacity,
                      const uint64_t* keys, uint64_t n, uint64_t* vals_out, uint8_t* found_out,
                      void* stream);
int pip_rt_delete_u64(uint64_t* table_keys, uint64_t capacity, const uint64_t* keys, uint64_t n,
                      void* workspace, size_t workspace_bytes, uint64_t* count_out, void* stream);

/* ---- rotate: strong.rotate (strong.py:67-95) ------------------------------ *
 * Left rotation: out[i] = in[(i + o) mod n], 0 <= o <= n.                   */
int pip_rotate_u64(uint64_t* a, uint64_t n, uint64_t o, void* scratch, size_t scratch_bytes,
                   void* stream);

/* In-place reversal of a[0:n) (strong.py:67-82, the rotation's step). */
int pip_reverse_u64(uint64_t* a, uint64_t n, void* stream);
/* memmove inside one device array: a[dst : dst+len) = the old a[src :
 * src+len).  Overlapping left moves run in ONE pass on the look-back
 * machinery (scratch as pip_filter_u64; pip_scratch_status applies);
 * disjoint ranges copy; overlapping right moves rotate a[src : dst+len).
 * The sharded filter's local shift (distributed.py).                       */
int pip_move_u64(uint64_t* a, uint64_t dst, uint64_t src, uint64_t len, void* scratch,
                 size_t scratch_bytes, void* stream);

/* ---- partition: strong.partition_unstable / relaxed.partition_relaxed ---- *
 * Unstable in-place partition (strong.py:394-419, relaxed.py:312-344): on
 * return a[0:m) holds the words with keep(x), a[m:n) the others (multiset
 * preserved); m is written to device m_dev.  workspace holds
 * pip_partition_workspace_bytes(n) (O(n/4096) descriptors).  Stream-ordered.
 * pip_partition_u64_host: same on a host array (synchronous).  Above one
 * host chunk (2^24 words) it is streamed: chunks are uploaded from both
 * ends, partitioned on the device one by one, and their kept / dropped
 * words written back to the front / back of the array as soon as the host
 * range they land in has been uploaded (the arrangement inside each side
 * differs from the device entry point's; the contract is the same).
 * PIP_PARTITION_HOST_INPLACE=1: upload all, device partition, copy back. */
size_t pip_partition_workspace_bytes(uint64_t n);
int pip_partition_u64(uint64_t* a, uint64_t n, const pip_pred* pred, uint64_t* m_dev,
                      void* workspace, size_t workspace_bytes, void* stream);
int pip_partition_u64_host(uint64_t* host_a, uint64_t n, const pip_pred* pred, uint64_t* m_out,
                           int device);

/* ---- one quicksort level: pip_partition_u64 over nseg disjoint segments
 * (strong.py:431-452, relaxed.py:347-369, one call per level of the
 * recursion instead of one per node).  Segment g = a[seg_lo[g] :
 * seg_lo[g] + seg_len[g]) is partitioned by (x kind operand[g]) with kind in
 * PIP_PRED_LT..PIP_PRED_EQ; its kept count goes to device m_dev[g].
 * seg_lo / seg_len / operand are HOST arrays; workspace holds
 * pip_partition_workspace_bytes(max seg_len).  Stream-ordered.            */
int pip_partition_segments_u64(uint64_t* a, const uint64_t* seg_lo, const uint64_t* seg_len,
                               const uint64_t* operand, uint32_t kind, uint64_t* m_dev,
                               uint64_t nseg, void* workspace, size_t workspace_bytes,
                               void* stream);

/* ---- quicksort leaves: the base case of strong.quicksort_strong /
 * relaxed.quicksort_relaxed (strong.py:453-454, relaxed.py:370-371):
 * sorts a[seg_lo[g] : seg_lo[g] + seg_len[g]) ascending (unsigned) for every
 * g < nseg; seg_len[g] <= 2^20, segments disjoint; device arrays.  The
 * recursion above it partitions with pip_partition_u64.                   */
int pip_sort_segments_u64(uint64_t* a, const uint64_t* seg_lo_dev, const uint32_t* seg_len_dev,
                          uint64_t nseg, void* stream);

/* pip_sort_segments_grid_u64: the same contract for segments of up to
 * 2^28 words; max_len >= every seg_len[g] (host value).  The network is
 * spread over the grid (one launch per stage wider than 8192 words), so a
 * few long segments still use every SM.                                   */
int pip_sort_segments_grid_u64(uint64_t* a, const uint64_t* seg_lo_dev, const uint32_t* seg_len_dev,
                               uint64_t nseg, uint64_t max_len, void* stream);

/* ---- list contraction / ranking: contraction.list_contract / list_rank ---- *
 * (contraction.py:264-365 on detres.run_rounds, detres.py:256-307).  next /
 * prev / p are device u64[n] (NIL = 2^64-1 ends a chain; p distinct
 * priorities); rounds of `prefix` = b(n) active ids with the reference's
 * structure, so committed_per_round_host[r] (host, r < rounds_cap) and
 * *rounds_out equal its RoundStats.  rank == 0: every element splices out
 * and keeps (prev, next) = its splice-time neighbours; trace_host (host
 * u64[n], NULL ok) receives the committed ids round by round, splice_host
 * (host u64[3n], NULL ok) the (v, u, x) triples (on_splice).  rank != 0:
 * list_rank — prev receives the 0-based ranks, next bookkeeping marks.
 * Synchronizes once per round.  PIP_ERR_LIVELOCK after 64 zero rounds.    */
size_t pip_list_contract_workspace_bytes(uint64_t n, uint64_t prefix, int rank);
int pip_list_contract_u64(uint64_t* next, uint64_t* prev, const uint64_t* p, uint64_t n,
                          uint64_t prefix, int rank, uint64_t* committed_per_round_host,
                          uint64_t rounds_cap, uint64_t* rounds_out, uint64_t* trace_host,
                          uint64_t* splice_host, void* workspace, size_t workspace_bytes,
                          void* stream);

/* ---- tree contraction, whole round loop: contraction.tree_contract
 * (contraction.py:368-559 on detres.run_rounds).  parent / left / right /
 * p / values: device u64[n] (NIL = 2^64-1), rewritten in place (values
 * folded with combine 0 add, 1 max, 2 min, 3 xor, mod 2^64).  The frontier
 * queue, sweep cursor, active list and rake-parent map live in `workspace`
 * (pip_tree_contract_workspace_bytes(n, prefix), O(prefix)); the host loop
 * reads a few counts per round.  HOST outputs: committed_per_round_host
 * [rounds_cap], trace_host (u64[n], NULL ok: committed ids per round in
 * packed order), roots_host (u64[2n]: (root, folded value) pairs, count in
 * *nroots_out), *violations_out (debug != 0: parent-child pairs contracted
 * together, contraction.py:481-485).  PIP_ERR_TABLE = frontier overflow,
 * PIP_ERR_LIVELOCK after 64 zero rounds.  Synchronizes.                    */
size_t pip_tree_contract_workspace_bytes(uint64_t n, uint64_t prefix);
int pip_tree_contract_u64(uint64_t* parent, uint64_t* left, uint64_t* right, const uint64_t* p,
                          uint64_t* values, uint64_t n, uint64_t prefix, int combine, int debug,
                          uint64_t* committed_per_round_host, uint64_t rounds_cap, uint64_t* rounds_out,
                          uint64_t* trace_host, uint64_t* roots_host, uint64_t* nroots_out,
                          uint64_t* violations_out, void* workspace, size_t workspace_bytes,
                          void* stream);

/* ---- tree contraction, one round step: contraction.tree_contract (contraction.py:368-559) *
 * The frontier queue / cursor bookkeeping (O(prefix) per round) is the
 * caller's; one call runs one device step of a round on the device-resident
 * forest (parent/left/right/p/values, NIL = 2^64-1):
 *   step 0: flags[v - lo] = contractible-when-swept, v in [lo, hi)
 *   step 1: flags[k] = eligibility of ids[k], k < fill (sorted_ids: the same
 *           ids ascending, for the active-neighbour test)
 *   step 2: gathered[6k..6k+5] = (parent, child, is_left, parent's child
 *           count, grandparent, value) of the committing ids[k] before any
 *           surgery
 *   step 3: fold values (combine 0 add, 1 max, 2 min, 3 xor; mod 2^64) and
 *           re-link, from step 2's gathered state.  Stream-ordered.        */
int pip_tree_round_u64(int step, uint64_t* parent, uint64_t* left, uint64_t* right,
                       const uint64_t* p, uint64_t* values, uint64_t lo, uint64_t hi,
                       const uint32_t* ids, uint64_t fill, const uint32_t* sorted_ids,
                       uint8_t* flags, uint64_t* gathered, int combine, void* stream);

/* ---- merge: strong.merge_strong / relaxed.merge_relaxed ------------------ *
 * a[0:split) and a[split:n) are sorted ascending (unsigned); on return a is
 * sorted.  `workspace`/`workspace_bytes` is the metered auxiliary space
 * (pip_merge_workspace_bytes tells how much a given budget can use); with
 * workspace_bytes == 0 the strong (zero-heap) schedule runs on scratch only.
 * check_sorted != 0 reproduces debug=True (PIP_ERR_UNSORTED).  `scratch`
 * (pip_scratch_bytes, required for n > 8192) holds the block phase's
 * per-CTA load-status words: O(#SMs), independent of n, unmetered.
 * Replaces strong.py:496-522 and relaxed.py:579-612.                        */
int pip_merge_u64(uint64_t* a, uint64_t n, uint64_t split, int check_sorted,
                  void* workspace, size_t workspace_bytes, void* scratch, size_t scratch_bytes,
                  void* stream);
/* device workspace (bytes) the relaxed merge uses for n, split and budget
 * b = budget_words (b(n) of the caller's EpsilonConfig); 0 = strong path. */
size_t pip_merge_workspace_bytes(uint64_t n, uint64_t split, uint64_t budget_words);
/* the same contract on a host array (synchronous).  Streamed: the output is
 * produced in chunks of 2^24 words (PIP_HOST_CHUNK_LOG2; the ring of
 * PIP_HOST_NBUF chunk buffers stays within budget_words when it is > 0),
 * each merged out of place on the device from the uploaded runs and copied
 * straight back, so uploads, merges and write-backs overlap; the host array
 * is still updated in place (every word is uploaded before the write-back
 * that overwrites it).  PIP_MERGE_HOST_INPLACE=1: upload all, in-place
 * device merge, copy back. */
int pip_merge_u64_host(uint64_t* host_a, uint64_t n, uint64_t split, uint64_t budget_words,
                       int device);
/* device workspace (bytes) pip_merge_u64_host uses besides its staging copy
 * of the array: the output ring (or, with PIP_MERGE_HOST_INPLACE=1, the
 * device merge's workspace) — what a relaxed caller charges to its meter. */
size_t pip_merge_host_workspace_bytes(uint64_t n, uint64_t split, uint64_t budget_words);

/* ---- random permutation: relaxed.random_permutation (relaxed.py:220-251) - *
 * Applies the Knuth swap sequence H (swap a[i], a[H[i]] for i = n-1..0) as
 * deterministic-reservation rounds over prefix = b(n) pending iterates
 * (detres.run_rounds, detres.py:256-307), with the reference's round
 * structure (descending ids, self-swaps retired at ingestion, failures
 * packed first), so rounds / committed-per-round / trace are identical.
 *   committed_per_round_host: HOST u64[rounds_cap] (NULL ok), written by the
 *   call as the rounds complete (it synchronizes)
 *   trace_dev: device u64[n_iterates] of committed ids in round/packed order
 *   (NULL ok); debug != 0 runs the clean-table sweep (relaxed.py:212-217).
 * workspace must hold pip_rp_workspace_bytes(n, prefix, variant).
 * stats_host receives the round statistics (the call synchronizes).        */
size_t pip_rp_workspace_bytes(uint64_t n, uint64_t prefix, int variant);
int pip_random_permutation_u64(uint64_t* a, const uint64_t* h, uint64_t n, uint64_t prefix,
                               int variant, int debug, uint64_t* committed_per_round_host,
                               uint64_t rounds_cap, uint64_t* trace_dev,
                               void* workspace, size_t workspace_bytes,
                               pip_rp_stats* stats_host, void* stream);
/* relaxed.validate_swap_sequence (relaxed.py:55-58) + the non-self count of
 * relaxed.py:239: nonself_dev receives #{i : H[i] != i}; returns
 * PIP_ERR_INVALID_SWAPS (after syncing) when some H[i] > i.               */
int pip_validate_swaps_u64(const uint64_t* h, uint64_t n, uint64_t* nonself_dev,
                           void* scratch, size_t scratch_bytes, void* stream);
int pip_random_permutation_u64_host(uint64_t* host_a, const uint64_t* host_h, uint64_t n,
                                    uint64_t prefix, int variant, pip_rp_stats* stats_host,
                                    int device);

/* ---- multi-GPU: sharded scan and filter on an NCCL communicator ----------- *
 * SURVEY.md 8(b) "multi-GPU variants taking an ncclComm_t plus shard
 * descriptors", 8(e).  The reference has no distributed code; these restate
 * distributed.py's sharded_scan / sharded_filter over the NCCL C API.  One
 * process per GPU; the global array of n_global words is split evenly, rank r
 * owning global [r*S, min(n_global, (r+1)*S)), S = ceil(n_global / world).
 * nccl_comm is an ncclComm_t of `world` ranks in which the caller is `rank`
 * (void* here: this header needs no nccl.h).  NCCL is resolved at run time
 * from the process's libnccl.so.2 (or PIP_NCCL_LIB): PIP_ERR_UNSUPPORTED when
 * none can be loaded, PIP_ERR_CUDA when an NCCL call fails.  workspace:
 * device memory of pip_sharded_workspace_bytes(world) = 8 (world + 2) bytes.
 *
 * pip_scan_u64_sharded: in-place scan of the GLOBAL array (strong.scan's
 * contract, strong.py:151-166) — local fold, allgather of the shard totals,
 * device carry, local scan with the carry; stream-ordered, no host
 * synchronization; total_dev (device, NULL ok) receives the global total.
 *
 * pip_filter_u64_sharded: stable filter of the GLOBAL array, in place
 * (strong.filter_kway's contract, strong.py:283-349): on return the packed
 * prefix global [0, m) holds the kept words in order, *m_out (HOST) = m and
 * *local_len_out (HOST, NULL ok) = how many words of that prefix sit in this
 * rank's shard (local [0, len)).  Local filter, allgather of the kept counts,
 * then pip_filter_shard_plan's moves: ncclSend of the head that lands in
 * lower shards, one in-place shift of the rest (pip_move_u64), ncclRecv of
 * the words of higher ranks into their final slots — destination precedes
 * source at rank granularity (strong.py:317-327).  Synchronizes (the plan
 * needs the counts on the host).  No rank holds a copy of its shard.
 *
 * pip_filter_shard_plan: the plan alone (host arithmetic, no GPU, no NCCL):
 * counts = HOST u64[world] kept words per shard; down / up receive at most
 * world - 1 pieces each.                                                    */
typedef struct pip_shard_piece {
  uint32_t peer;          /* rank the piece goes to (down) / comes from (up) */
  uint32_t reserved;
  uint64_t local_offset;  /* word offset inside the caller's shard */
  uint64_t length;        /* words */
} pip_shard_piece;
size_t pip_sharded_workspace_bytes(int world);
int pip_nccl_available(void); /* 1 when the NCCL entry points resolved */
int pip_scan_u64_sharded(uint64_t* a_local, uint64_t n_local, int op, uint64_t init, int inclusive,
                         void* nccl_comm, int rank, int world, void* workspace,
                         size_t workspace_bytes, uint64_t* total_dev, void* scratch,
                         size_t scratch_bytes, void* stream);
int pip_filter_shard_plan(const uint64_t* counts, int world, int rank, uint64_t n_global,
                          pip_shard_piece* down, int* n_down, uint64_t* stay_src,
                          uint64_t* stay_len, pip_shard_piece* up, int* n_up);
int pip_filter_u64_sharded(uint64_t* a_local, uint64_t n_local, uint64_t n_global,
                           const pip_pred* pred, void* nccl_comm, int rank, int world,
                           void* workspace, size_t workspace_bytes, uint64_t* m_out,
                           uint64_t* local_len_out, void* scratch, size_t scratch_bytes,
                           void* stream);

/* ---- input generation (runtime.Rng, runtime.py:263-302) ------------------ *
 * out[k] = mix64(seed + (lo + k + 1) * GOLDEN) >> shift   (Rng.words)
 * swaps: out[k] = Rng.words(lo..)[k] % (lo + k + 1)      (make_swap_sequence) */
int pip_rng_words_u64(uint64_t* out, uint64_t lo, uint64_t count, uint64_t seed,
                      uint32_t shift, void* stream);
int pip_make_swaps_u64(uint64_t* out, uint64_t lo, uint64_t count, uint64_t seed,
                       void* stream);

/* ---- microbenchmarks used by the roofline (bench.py) --------------------- */
/* iters rounds of 8-byte read-modify-write at uniform random word indices of
 * buf[0:n) (one per thread of a full grid); returns device time in ms. */
int pip_bench_random_rmw(uint64_t* buf, uint64_t n, uint64_t updates, uint64_t seed,
                         float* ms_out, void* stream);
/* the same with the request form chosen: 0 load + store (two requests per
 * update), 1 atomic exchange whose old value is consumed (the form the
 * permutation's swaps take above 2^28 words), 2 reduction (no return). */
int pip_bench_random_update(uint64_t* buf, uint64_t n, uint64_t updates, uint64_t seed, int form,
                            float* ms_out, void* stream);

#ifdef __cplusplus
}
#endif
#endif /* PIP_H_ */
