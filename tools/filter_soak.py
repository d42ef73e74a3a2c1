"""Back-to-back full-size filters with the stall status read after every call."""
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
desc = pip.pred.mod_eq(3, 0).descriptor()
worst, m0 = 0.0, None
for r in range(reps):
    pip.Rng(1).words_device(0, n, shift=1, out=a)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    rc = lib.pip_filter_u64(a.data_ptr(), n, C.byref(desc), out.data_ptr(), sp, sb, st)
    stall = lib.pip_scratch_status(sp, st)
    dt = (time.perf_counter() - t0) * 1e3
    m = int(out.item())
    m0 = m if m0 is None else m0
    worst = max(worst, dt)
    if rc or stall or dt > 100 or m != m0:
        print(f"rep {r}: rc={rc} stall={stall} m={m} {dt:.1f} ms", flush=True)
print(f"done {reps} reps of 2^{lg}, m={m0}, worst {worst:.2f} ms", flush=True)
