"""Back-to-back full-size scans with the stall status read after every call
(soak test of the look-back pipeline; PIP_SCAN_CFG / PIP_LB_STRIDE select the shape)."""
import ctypes as C
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch  # noqa: E402

import paper_2103_01216_b200 as pip  # noqa: E402

lg = int(sys.argv[1]) if len(sys.argv) > 1 else 32
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 30
lib = pip._lib.load()
n = 1 << lg
st = torch.cuda.current_stream().cuda_stream
sp, sb = pip.runtime.scratch_for(0, st)
a = torch.empty(n, dtype=torch.int64, device="cuda")
out = torch.zeros(1, dtype=torch.int64, device="cuda")
pip.Rng(1).words_device(0, n, shift=44, out=a)
worst = 0.0
for r in range(reps):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    rc = lib.pip_scan_u64(a.data_ptr(), n, 0, 0, 1, out.data_ptr(), sp, sb, st)
    stall = lib.pip_scratch_status(sp, st)
    dt = (time.perf_counter() - t0) * 1e3
    worst = max(worst, dt)
    if rc or stall or dt > 100:
        print(f"rep {r}: rc={rc} stall={stall} {dt:.1f} ms", flush=True)
print(f"done {reps} reps of 2^{lg}, worst {worst:.2f} ms", flush=True)
