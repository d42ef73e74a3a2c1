"""Random 8-byte RMW rate vs the size of the region the indices fall in
(pip_bench_random_rmw): does address locality help the random accesses?"""
import ctypes as C
import json
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch  # noqa: E402

import paper_2103_01216_b200 as pip  # noqa: E402

lib = pip._lib.load()
buf = torch.zeros(1 << 30, dtype=torch.int64, device="cuda")
st = torch.cuda.current_stream().cuda_stream
for lg in (20, 22, 24, 25, 26, 27, 28, 30):
    n = 1 << lg
    ms = C.c_float(0)
    upd = 1 << 28
    lib.pip_bench_random_rmw(buf.data_ptr(), n, upd, 7, C.byref(ms), st)  # warm
    lib.pip_bench_random_rmw(buf.data_ptr(), n, upd, 7, C.byref(ms), st)
    print(json.dumps({"region_words": n, "region_MB": n * 8 / 2**20, "updates": upd,
                      "ms": ms.value, "G_rmw_per_s": upd / (ms.value / 1e3) / 1e9}), flush=True)
