/*
 * pip_oracle.c — CPU restatement of the reference's hot path.
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and
 * bench.py's cpu_baseline / --impl reference legs may load this library, and
 * only as the checker or the timed CPU baseline — never on the product path
 * (the product is libpip.so, which has no CPU fallback).
 *
 * Parity pinning: every function is cross-checked in tests/ against the
 * reference `pipal` (imported from /root/reference/pkg/src in the build
 * container) and against golden fixtures generated from it
 * (tests/golden/make_golden.py).
 *
 * Two families:
 *   oracle_seq_*  sequential oracles, restating pkg/src/pipal/baselines.py
 *   oracle_ref_*  ports of the reference's own in-place algorithms
 *                 (strong.py / relaxed.py / detres.py), parallelised with
 *                 OpenMP the way the reference's fork-join pool intends;
 *                 these are the CPU baseline timed by bench.py.
 * Values are uint64 words; sums wrap mod 2^64; comparisons are unsigned.
 */
#include <omp.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

typedef uint64_t u64;
typedef uint32_t u32;

#define OP_ADD 0
#define OP_MAX 1
#define OP_MIN 2
#define OP_XOR 3

static inline u64 apply_op(int op, u64 a, u64 b) {
  switch (op) {
    case OP_MAX: return a > b ? a : b;
    case OP_MIN: return a < b ? a : b;
    case OP_XOR: return a ^ b;
    default: return a + b;
  }
}
static inline u64 op_identity(int op) { return op == OP_MIN ? ~0ull : 0ull; }

/* ------------------------------------------------------------------------
 * predicates (include/pip.h pip_pred semantics)                           */
enum { P_ALL = 0, P_MASK_EQ, P_MOD_EQ, P_LT, P_LE, P_GT, P_GE, P_EQ };
static inline int pred_eval(u32 kind, u32 negate, u64 a, u64 b, u64 x) {
  int r;
  switch (kind) {
    case P_MASK_EQ: r = (x & a) == b; break;
    case P_MOD_EQ: r = (x % a) == b; break;
    case P_LT: r = x < a; break;
    case P_LE: r = x <= a; break;
    case P_GT: r = x > a; break;
    case P_GE: r = x >= a; break;
    case P_EQ: r = x == a; break;
    default: r = 1; break;
  }
  return negate ? !r : r;
}

/* ========================================================================
 * Sequential oracles (baselines.py)
 * ======================================================================== */

/* baselines.py:26-35 seq_scan: exclusive prefix sums mod 2^64 + total.
 * Generalised to strong.scan's `op` path (strong.py:132-148, 157-166):
 * exclusive a[i] = op(init, x0..x_{i-1}), a[0] = init; inclusive adds x_i;
 * total = fold of all x (without init). */
void oracle_seq_scan(const u64* in, u64* out, u64 n, int op, u64 init, int inclusive, u64* total) {
  u64 run = op_identity(op);
  for (u64 i = 0; i < n; ++i) {
    const u64 x = in[i];
    if (inclusive) {
      run = apply_op(op, run, x);
      out[i] = apply_op(op, init, run);
    } else {
      out[i] = apply_op(op, init, run);
      run = apply_op(op, run, x);
    }
  }
  if (total) *total = run;
}

/* baselines.py:38-41 seq_filter: stable filter into a fresh array */
u64 oracle_seq_filter(const u64* in, u64 n, u32 kind, u32 negate, u64 pa, u64 pb, u64* out) {
  u64 m = 0;
  for (u64 i = 0; i < n; ++i)
    if (pred_eval(kind, negate, pa, pb, in[i])) out[m++] = in[i];
  return m;
}

/* baselines.py:44-54 seq_knuth_shuffle: for i = n-1 .. 0 swap a[i], a[h[i]] */
void oracle_seq_knuth_shuffle(u64* a, const u64* h, u64 n) {
  for (u64 k = n; k-- > 0;) {
    const u64 j = h[k];
    const u64 t = a[k];
    a[k] = a[j];
    a[j] = t;
  }
}

/* baselines.py:99-114 seq_two_finger_merge (ties taken from x) */
void oracle_seq_merge(const u64* x, u64 nx, const u64* y, u64 ny, u64* out) {
  u64 i = 0, j = 0, k = 0;
  while (i < nx && j < ny) out[k++] = (x[i] <= y[j]) ? x[i++] : y[j++];
  while (i < nx) out[k++] = x[i++];
  while (j < ny) out[k++] = y[j++];
}

/* ========================================================================
 * Ports of the reference's in-place algorithms (CPU baseline)
 * ======================================================================== */

#define SCAN_BASE 256
#define TASK_GRAIN (1 << 16)

/* strong.py:107-115 _up_sweep_add (inclusive positions [s, t]) */
static void up_sweep_add(u64* a, u64 s, u64 t) {
  if (t - s + 1 <= SCAN_BASE) {
    for (u64 i = s + 1; i <= t; ++i) a[i] += a[i - 1];
    return;
  }
  const u64 mid = s + (t - s) / 2;
  if (t - s > TASK_GRAIN) {
#pragma omp task
    up_sweep_add(a, s, mid);
    up_sweep_add(a, mid + 1, t);
#pragma omp taskwait
  } else {
    up_sweep_add(a, s, mid);
    up_sweep_add(a, mid + 1, t);
  }
  a[t] += a[mid];
}

/* strong.py:118-129 _down_sweep_add */
static void down_sweep_add(u64* a, u64 s, u64 t, u64 p) {
  if (t - s + 1 <= SCAN_BASE) {
    u64 prev = a[s];
    a[s] = p;
    for (u64 i = s + 1; i <= t; ++i) {
      const u64 cur = a[i];
      a[i] = prev + p;
      prev = cur;
    }
    return;
  }
  const u64 mid = s + (t - s) / 2;
  const u64 left = a[mid];
  if (t - s > TASK_GRAIN) {
#pragma omp task
    down_sweep_add(a, s, mid, p);
    down_sweep_add(a, mid + 1, t, p + left);
#pragma omp taskwait
  } else {
    down_sweep_add(a, s, mid, p);
    down_sweep_add(a, mid + 1, t, p + left);
  }
}

/* strong.py:151-166 scan (op=None): exclusive in-place scan, returns total */
u64 oracle_ref_scan(u64* a, u64 n, int threads) {
  if (n == 0) return 0;
  u64 total = 0;
#pragma omp parallel num_threads(threads)
#pragma omp single
  {
    up_sweep_add(a, 0, n - 1);
    total = a[n - 1];
    down_sweep_add(a, 0, n - 1, 0);
  }
  return total;
}

/* strong.py:296-349 filter_kway (sqrt(n) chunks, batches of <= 256 chunks
 * whose destinations precede the batch's first source) */
static u64 compact_chunk(u64* a, u64 s, u64 e, u32 kind, u32 neg, u64 pa, u64 pb) {
  u64 w = s;
  for (u64 i = s; i < e; ++i)
    if (pred_eval(kind, neg, pa, pb, a[i])) a[w++] = a[i];
  return w - s;
}
u64 oracle_ref_filter_kway(u64* a, u64 n, u32 kind, u32 neg, u64 pa, u64 pb, int threads) {
  if (n == 0) return 0;
  u64 k = 1;
  while (k * k < n) ++k; /* ceil(sqrt(n)) as math.isqrt + 1 */
  {
    u64 r = 0;
    while ((r + 1) * (r + 1) <= n) ++r;
    k = (r * r < n) ? r + 1 : r;
  }
  const u64 chunk = (n + k - 1) / k;
  const u64 nchunks = (n + chunk - 1) / chunk;
  u64 m = 0, c = 0;
  u64 counts[256], csum[257];
  while (c < nchunks) {
    const u64 jcap = (nchunks - c) < 256 ? (nchunks - c) : 256;
#pragma omp parallel for num_threads(threads) schedule(dynamic, 1)
    for (u64 t = 0; t < jcap; ++t) {
      const u64 s = (c + t) * chunk, e = (s + chunk < n) ? s + chunk : n;
      u64 cnt = 0;
      for (u64 i = s; i < e; ++i) cnt += pred_eval(kind, neg, pa, pb, a[i]);
      counts[t] = cnt;
    }
    csum[0] = 0;
    for (u64 t = 0; t < jcap; ++t) csum[t + 1] = csum[t] + counts[t];
    const u64 first_src = c * chunk;
    u64 lo = 1, hi = jcap;
    while (lo < hi) {
      const u64 mid = (lo + hi + 1) / 2;
      if (m + csum[mid] <= first_src) lo = mid; else hi = mid - 1;
    }
    const u64 j = (m + csum[lo] <= first_src) ? lo : 0;
    if (j == 0) {
      const u64 s = c * chunk, e = (s + chunk < n) ? s + chunk : n;
      const u64 cnt = compact_chunk(a, s, e, kind, neg, pa, pb);
      if (m != s) memmove(a + m, a + s, cnt * 8);
      m += cnt;
      c += 1;
      continue;
    }
#pragma omp parallel for num_threads(threads) schedule(dynamic, 1)
    for (u64 t = 0; t < j; ++t) {
      const u64 s = (c + t) * chunk, e = (s + chunk < n) ? s + chunk : n;
      const u64 cnt = compact_chunk(a, s, e, kind, neg, pa, pb);
      const u64 dst = m + csum[t];
      if (dst != s) memmove(a + dst, a + s, cnt * 8);
    }
    m += csum[j];
    c += j;
  }
  return m;
}

/* strong.py:67-95 rotate by triple reversal */
static void reverse_range(u64* a, u64 s, u64 t) {
  while (t > s + 1) {
    --t;
    const u64 x = a[s];
    a[s] = a[t];
    a[t] = x;
    ++s;
  }
}
static void rotate_range(u64* a, u64 s, u64 t, u64 o) {
  if (o == 0 || o == t - s || t - s < 2) return;
  reverse_range(a, s, s + o);
  reverse_range(a, s + o, t);
  reverse_range(a, s, t);
}
void oracle_ref_rotate(u64* a, u64 n, u64 o) { rotate_range(a, 0, n, o); }

/* strong.py:352-419 partition_unstable: blocks of SCRATCH_WORDS (256)
 * partitioned through a scratch copy (true words first, both sides in
 * order, :352-363), true prefixes folded leftward by range swaps (:366-373)
 * or rotations (:376-391); outer chunks of max(ceil(n / ceil(sqrt n)), 256)
 * words folded the same way (:394-419).  Sequential, like the reference. */
#define PART_SCRATCH 256
static u64 block_partition(u64* a, u64 s, u64 e, u32 kind, u32 neg, u64 pa, u64 pb) {
  u64 tmp[PART_SCRATCH];
  const u64 len = e - s;
  u64 t = 0;
  for (u64 i = 0; i < len; ++i) t += pred_eval(kind, neg, pa, pb, a[s + i]);
  if (t == len) return t;
  memcpy(tmp, a + s, len * 8);
  u64 wt = s, wf = s + t;
  for (u64 i = 0; i < len; ++i) {
    if (pred_eval(kind, neg, pa, pb, tmp[i])) a[wt++] = tmp[i];
    else a[wf++] = tmp[i];
  }
  return t;
}
static void swap_ranges(u64* a, u64 p, u64 q, u64 cnt) {
  for (u64 i = 0; i < cnt; ++i) {
    const u64 x = a[p + i];
    a[p + i] = a[q + i];
    a[q + i] = x;
  }
}
static u64 partition_range(u64* a, u64 lo, u64 hi, u32 kind, u32 neg, u64 pa, u64 pb) {
  u64 w = lo, s = lo;
  while (s < hi) {
    const u64 e = (s + PART_SCRATCH < hi) ? s + PART_SCRATCH : hi;
    const u64 t = block_partition(a, s, e, kind, neg, pa, pb);
    if (t) {
      if (w + t <= s) swap_ranges(a, w, s, t);
      else if (w < s) rotate_range(a, w, s + t, s - w);
      w += t;
    }
    s = e;
  }
  return w - lo;
}
u64 oracle_ref_partition_unstable(u64* a, u64 n, u32 kind, u32 neg, u64 pa, u64 pb) {
  if (n == 0) return 0;
  u64 r = 0;
  while ((r + 1) * (r + 1) <= n) ++r;
  const u64 k = (r * r < n) ? r + 1 : r;
  u64 chunk = (n + k - 1) / k;
  if (chunk < PART_SCRATCH) chunk = PART_SCRATCH;
  u64 m = 0, s = 0;
  while (s < n) {
    const u64 e = (s + chunk < n) ? s + chunk : n;
    const u64 t = partition_range(a, s, e, kind, neg, pa, pb);
    if (t) {
      if (m + t <= s) swap_ranges(a, m, s, t);
      else if (m < s) rotate_range(a, m, s + t, s - m);
      m += t;
    }
    s = e;
  }
  return m;
}

/* strong.py:474-488 _split_point */
static u64 split_point(const u64* a, u64 lo, u64 mid, u64 hi, u64 h) {
  const u64 na = mid - lo, nb = hi - mid;
  u64 ilo = h > nb ? h - nb : 0, ihi = na < h ? na : h;
  while (ilo < ihi) {
    const u64 im = (ilo + ihi) / 2, jm = h - im;
    if (jm > 0 && im < na && a[mid + jm - 1] >= a[lo + im]) ilo = im + 1;
    else ihi = im;
  }
  return ilo;
}
/* strong.py:462-471 _merge_base (<= 256 words) */
static void merge_base(u64* a, u64 lo, u64 mid, u64 hi) {
  u64 tmp[256];
  const u64 len = hi - lo;
  memcpy(tmp, a + lo, len * 8);
  oracle_seq_merge(tmp, mid - lo, tmp + (mid - lo), hi - mid, a + lo);
}
static void merge_rec(u64* a, u64 lo, u64 mid, u64 hi) {
  const u64 na = mid - lo, nb = hi - mid;
  if (na == 0 || nb == 0) return;
  if (hi - lo <= 256) {
    merge_base(a, lo, mid, hi);
    return;
  }
  const u64 h = (hi - lo) / 2;
  const u64 i = split_point(a, lo, mid, hi, h), j = h - i;
  rotate_range(a, lo + i, mid + j, mid - (lo + i));
  const u64 cut = lo + h;
  if (hi - lo > TASK_GRAIN) {
#pragma omp task
    merge_rec(a, lo, lo + i, cut);
    merge_rec(a, cut, mid + j, hi);
#pragma omp taskwait
  } else {
    merge_rec(a, lo, lo + i, cut);
    merge_rec(a, cut, mid + j, hi);
  }
}
/* strong.py:496-522 merge_strong */
void oracle_ref_merge_strong(u64* a, u64 n, u64 split, int threads) {
#pragma omp parallel num_threads(threads)
#pragma omp single
  merge_rec(a, 0, split, n);
}

/* ------------------------------------------------------------------------
 * relaxed.py:64-251 random_permutation on detres.py:256-307 run_rounds.
 * Same round structure as the reference (descending ids from a window,
 * self-swaps skipped, failures packed first, write-max reservations; the
 * `final` variant serves the fresh id range from a dense array).
 * Returns 0, or 3 on livelock, 2 on invalid H, 7 if n >= 2^32 - 1.       */
#define V_NAIVE 0
#define V_FLAT 1
#define V_ONERES 2
#define V_FINAL 3
static const u64 GOLDEN = 0x9E3779B97F4A7C15ull;
static const u64 T_EMPTY = ~0ull;

typedef struct {
  u64* w;
  u32 logcap;
  u64 claims;
} table_t;

static inline u64 t_home(const table_t* t, u32 key) { return ((u64)key * GOLDEN) >> (64 - t->logcap); }

static u64 t_reserve(table_t* t, u32 key, u32 val) {
  const u64 mask = (1ull << t->logcap) - 1, want = ((u64)key << 32) | val;
  u64 s = t_home(t, key);
  for (;;) {
    u64 cur = __atomic_load_n(&t->w[s], __ATOMIC_RELAXED);
    if (cur == T_EMPTY) {
      u64 exp = T_EMPTY;
      if (__atomic_compare_exchange_n(&t->w[s], &exp, want, 0, __ATOMIC_RELAXED, __ATOMIC_RELAXED)) {
        __atomic_fetch_add(&t->claims, 1, __ATOMIC_RELAXED);
        return s;
      }
      cur = exp;
    }
    if ((u32)(cur >> 32) == key) {
      while ((u32)cur < val &&
             !__atomic_compare_exchange_n(&t->w[s], &cur, want, 0, __ATOMIC_RELAXED, __ATOMIC_RELAXED)) {
      }
      return s;
    }
    s = (s + 1) & mask;
  }
}
static int t_lookup(const table_t* t, u32 key, u32* val) {
  const u64 mask = (1ull << t->logcap) - 1;
  u64 s = t_home(t, key);
  for (;;) {
    const u64 cur = t->w[s];
    if (cur == T_EMPTY) return 0;
    if ((u32)(cur >> 32) == key) {
      *val = (u32)cur;
      return 1;
    }
    s = (s + 1) & mask;
  }
}
static inline void atomic_max_u32(u32* p, u32 v) {
  u32 cur = __atomic_load_n(p, __ATOMIC_RELAXED);
  while (cur < v && !__atomic_compare_exchange_n(p, &cur, v, 0, __ATOMIC_RELAXED, __ATOMIC_RELAXED)) {
  }
}

int oracle_ref_random_permutation(u64* a, const u64* h, u64 n, u64 prefix, int variant,
                                  u64* counts, u64 counts_cap, u64* trace, u64* rounds_out,
                                  u64* peak_out, u64* cap_out, int threads) {
  if (n >= 0xffffffffull) return 7;
  u64 n_iter = 0;
  for (u64 i = 0; i < n; ++i) {
    if (h[i] > i) return 2;
    n_iter += h[i] != i;
  }
  const int two_res = variant == V_NAIVE || variant == V_FLAT;
  u64 cap = 8;
  while (cap < (two_res ? 4 * prefix : 2 * prefix)) cap <<= 1;
  u32 logcap = 0;
  while ((1ull << logcap) < cap) ++logcap;
  if (cap_out) *cap_out = cap;
  *rounds_out = 0;
  if (peak_out) *peak_out = 0;
  if (n == 0 || n_iter == 0) return 0;
  const u64 P = prefix < n_iter ? prefix : n_iter; /* detres.py:267 */
  const u64 span_cap = prefix + prefix / 4 + 8;  /* relaxed.py:88 */
  table_t T = {(u64*)malloc(cap * 8), logcap, 0};
  memset(T.w, 0xff, cap * 8);
  u32* dense = (u32*)calloc(span_cap, 4);
  u32* ids = (u32*)malloc(P * 4);
  u32* tg = (u32*)malloc(P * 4);
  u32* slot = (u32*)malloc(P * 4);
  unsigned char* com = (unsigned char*)malloc(P);
  long long cursor = (long long)n - 1;
  u64 fill = 0, rounds = 0, zero = 0, tpos = 0, peak = 0;
  int rc = 0;
  for (;;) {
    /* refill: relaxed.py:107-120 next_ids */
    const u64 new_pos0 = fill;
    u64 count = P - fill;
    while (count > 0 && cursor >= 0) {
      const u64 hi = (u64)cursor;
      const u64 W = variant == V_FINAL ? span_cap : (count > 1024 ? count : 1024);
      const u64 lo = hi + 1 >= W ? hi + 1 - W : 0;
      u64 got = 0;
      for (u64 q = 0; q <= hi - lo && got < count; ++q) {
        const u64 id = hi - q;
        if (h[id] != id) {
          ids[fill + got] = (u32)id;
          tg[fill + got] = (u32)h[id];
          ++got;
        }
      }
      if (got) {
        cursor = (long long)ids[fill + got - 1] - 1;
        fill += got;
        break;
      }
      cursor = (long long)lo - 1;
    }
    if (fill == 0) break;
    u64 dlo = 1, dhi = 0;
    if (fill > new_pos0) {
      dhi = ids[new_pos0];
      dlo = ids[fill - 1];
    }
    /* reserve: relaxed.py:130-159 */
    T.claims = 0;
#pragma omp parallel for num_threads(threads) schedule(static)
    for (u64 k = 0; k < fill; ++k) {
      const u32 i = ids[k], t = tg[k];
      if (variant == V_FINAL && t >= dlo && t <= dhi) {
        atomic_max_u32(&dense[dhi - t], i + 1u);
        slot[k] = 0xffffffffu;
      } else {
        if (two_res) t_reserve(&T, i, i);
        slot[k] = (u32)t_reserve(&T, t, i);
      }
    }
    if (T.claims > peak) peak = T.claims;
    /* commit + swap: relaxed.py:161-197 */
    u64 ncommit = 0;
#pragma omp parallel for num_threads(threads) schedule(static) reduction(+ : ncommit)
    for (u64 k = 0; k < fill; ++k) {
      const u32 i = ids[k], t = tg[k];
      u32 v = 0;
      int own, tgt;
      if (variant == V_FINAL && k >= new_pos0) {
        const u32 dv = dense[dhi - i];
        own = dv == 0 || dv == i + 1u;
      } else if (two_res) {
        own = t_lookup(&T, i, &v) && v == i;
      } else {
        own = !t_lookup(&T, i, &v) || v == i;
      }
      if (variant == V_FINAL && t >= dlo && t <= dhi) tgt = dense[dhi - t] == i + 1u;
      else tgt = ((u32)T.w[slot[k]]) == i;
      com[k] = (unsigned char)(own && tgt);
      if (com[k]) {
        const u64 x = a[i];
        a[i] = a[t];
        a[t] = x;
        ncommit += 1;
      }
    }
    /* clean: relaxed.py:199-217 */
    memset(T.w, 0xff, cap * 8);
    if (variant == V_FINAL && dhi >= dlo) memset(dense, 0, (dhi - dlo + 1) * 4);
    if (rounds < counts_cap && counts) counts[rounds] = ncommit;
    if (trace)
      for (u64 k = 0; k < fill; ++k)
        if (com[k]) trace[tpos++] = ids[k];
    rounds += 1;
    if (ncommit == 0) {
      if (++zero >= 64) {
        rc = 3;
        break;
      }
      continue;
    }
    zero = 0;
    /* compact_by_mask(ids, ~committed): failures first, in order */
    u64 w = 0;
    for (u64 k = 0; k < fill; ++k)
      if (!com[k]) {
        ids[w] = ids[k];
        tg[w] = tg[k];
        ++w;
      }
    fill = w;
  }
  *rounds_out = rounds;
  if (peak_out) *peak_out = peak;
  free(T.w);
  free(dense);
  free(ids);
  free(tg);
  free(slot);
  free(com);
  return rc;
}

int oracle_max_threads(void) { return omp_get_max_threads(); }
