"""Time the host-buffer scan entry point on pinned memory (e2e tuning)."""
import ctypes as C, sys, time
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch
import paper_2103_01216_b200 as pip
lib = pip._lib.load()
n = 1 << (int(sys.argv[1]) if len(sys.argv) > 1 else 32)
h = torch.empty(n, dtype=torch.int64, pin_memory=True)
out = C.c_uint64()
tot = 0.0
for it in range(3):
    h.fill_(1)
    t1 = time.perf_counter()
    lib.pip_scan_u64_host(h.data_ptr(), n, 0, 0, 1, C.byref(out), 0)
    if it:
        tot += time.perf_counter() - t1
print(f"e2e {2 * n / tot / 1e9:.3f} G words/s ({16 * n * 2 / tot / 1e9:.1f} GB/s both directions)")
