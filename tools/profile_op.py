"""Run one hot-path op a few times at a chosen size (for ncu captures).

usage: python tools/profile_op.py --op scan --log2n 28 [--reps 3]
The op is called through the C ABI exactly as bench.py does; the last call
is the one to capture (ncu -k regex:<kernel> -s <reps-1> -c 1).
"""
import argparse
import ctypes as C
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))

import torch  # noqa: E402

import paper_2103_01216_b200 as pip  # noqa: E402
from bench import sort_run  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--op", default="scan")
ap.add_argument("--log2n", type=int, default=28)
ap.add_argument("--reps", type=int, default=3)
args = ap.parse_args()
lib = pip._lib.load()
n = 1 << args.log2n
st = torch.cuda.current_stream().cuda_stream
sp, sb = pip.runtime.scratch_for(0, st)
a = torch.empty(n, dtype=torch.int64, device="cuda")
out = torch.zeros(4, dtype=torch.int64, device="cuda")
if args.op == "scan":
    pip.Rng(1).words_device(0, n, shift=44, out=a)
    for _ in range(args.reps):
        assert lib.pip_scan_u64(a.data_ptr(), n, 0, 0, 1, out.data_ptr(), sp, sb, st) == 0
elif args.op == "filter":
    desc = pip.pred.mod_eq(3, 0).descriptor()
    for _ in range(args.reps):
        pip.Rng(1).words_device(0, n, shift=1, out=a)
        assert lib.pip_filter_u64(a.data_ptr(), n, C.byref(desc), out.data_ptr(), sp, sb, st) == 0
elif args.op == "merge":
    na = n // 2
    wb = lib.pip_merge_workspace_bytes(n, na, pip.EpsilonConfig(0.5).prefix_words(n))
    ws = torch.empty(wb, dtype=torch.uint8, device="cuda")
    for _ in range(args.reps):
        pip.Rng(1).words_device(0, n, shift=34, out=a)
        sort_run(a[:na], torch, pip)
        sort_run(a[na:], torch, pip)
        assert lib.pip_merge_u64(a.data_ptr(), n, na, 0, ws.data_ptr(), wb, sp, sb, st) == 0
elif args.op == "rp":
    h = pip.Rng(1).swaps_device(0, n)
    a = torch.arange(n, dtype=torch.int64, device="cuda")
    prefix = pip.EpsilonConfig(0.5).prefix_words(n)
    wb = lib.pip_rp_workspace_bytes(n, prefix, 3)
    ws = torch.empty(wb, dtype=torch.uint8, device="cuda")
    stats = pip._lib.PipRpStats()
    for _ in range(args.reps):
        assert lib.pip_random_permutation_u64(a.data_ptr(), h.data_ptr(), n, prefix, 3, 0, None, 0,
                                              None, ws.data_ptr(), wb, C.byref(stats), st) == 0
elif args.op == "rmw":
    # the permutation's roofline denominator: random 8-byte read-modify-writes
    # over an array of the C4 size (bench.py run_rp)
    ms = C.c_float(0)
    for _ in range(args.reps):
        assert lib.pip_bench_random_rmw(a.data_ptr(), n, n, 7, C.byref(ms), st) == 0
    print("rmw", n, "updates in", ms.value, "ms ->", n / (ms.value / 1e3) / 1e9, "G RMW/s")
elif args.op == "rmwx":
    # the same updates as one atomic exchange each (the form the swaps take above 2^28 words)
    ms = C.c_float(0)
    for _ in range(args.reps):
        assert lib.pip_bench_random_update(a.data_ptr(), n, n, 7, 1, C.byref(ms), st) == 0
    print("rmwx", n, "updates in", ms.value, "ms ->", n / (ms.value / 1e3) / 1e9, "G exchanges/s")
torch.cuda.synchronize()
print("ok", args.op, n)
