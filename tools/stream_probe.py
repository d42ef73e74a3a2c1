"""Streaming-rate probe: device time of reduce / count / scan / filter / torch copy at 2^k words.

usage: python tools/stream_probe.py [--log2n 32] [--reps 5]
Measurement aid for the roofline discussion in DESIGN.md; not part of the product.
"""
import argparse
import ctypes as C
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch  # noqa: E402

import paper_2103_01216_b200 as pip  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--log2n", type=int, default=32)
ap.add_argument("--reps", type=int, default=5)
args = ap.parse_args()
lib = pip._lib.load()
n = 1 << args.log2n
st = torch.cuda.current_stream().cuda_stream
sp, sb = pip.runtime.scratch_for(0, st)
a = torch.empty(n, dtype=torch.int64, device="cuda")
pip.Rng(1).words_device(0, n, shift=44, out=a)
out = torch.zeros(4, dtype=torch.int64, device="cuda")
desc = pip.pred.mod_eq(3, 0).descriptor()


def timed(fn, bytes_per_elem):
    fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(args.reps):
        fn()
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / args.reps
    return ms, bytes_per_elem * n / ms / 1e6


res = {}
res["reduce"] = timed(lambda: lib.pip_reduce_u64(a.data_ptr(), n, 0, out.data_ptr(), sp, sb, st), 8)
res["count"] = timed(lambda: lib.pip_count_u64(a.data_ptr(), n, C.byref(desc), out.data_ptr(), sp, sb, st), 8)
res["scan"] = timed(lambda: lib.pip_scan_u64(a.data_ptr(), n, 0, 0, 1, out.data_ptr(), sp, sb, st), 16)
b = torch.empty_like(a)
res["torch_copy"] = timed(lambda: b.copy_(a), 16)
del b
res["filter(scan input)"] = timed(lambda: lib.pip_filter_u64(a.data_ptr(), n, C.byref(desc), out.data_ptr(), sp, sb, st), 8 + 8 / 3)
for k, (ms, gbs) in res.items():
    print(f"{k:20s} {ms:8.3f} ms  {gbs:8.1f} GB/s")
