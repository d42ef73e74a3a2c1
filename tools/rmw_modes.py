"""Random 8-byte update rate over 8 GiB by request form (PIP_RMW_MODE):
0 load + store, 1 atomic exchange with the old value consumed, 2 reduction."""
import ctypes as C
import json
import os
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch  # noqa: E402

import paper_2103_01216_b200 as pip  # noqa: E402

lib = pip._lib.load()
buf = torch.zeros(1 << 30, dtype=torch.int64, device="cuda")
st = torch.cuda.current_stream().cuda_stream
for mode in (0, 1, 2, 0, 1, 2):
    os.environ["PIP_RMW_MODE"] = str(mode)
    ms = C.c_float(0)
    upd = 1 << 30
    lib.pip_bench_random_rmw(buf.data_ptr(), 1 << 30, upd, 7, C.byref(ms), st)
    print(json.dumps({"mode": mode, "updates": upd, "ms": ms.value,
                      "G_per_s": upd / (ms.value / 1e3) / 1e9}), flush=True)
