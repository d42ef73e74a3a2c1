"""Random-access rate vs the L2 fetch granularity hint
(cudaLimitMaxL2FetchGranularity): the random-RMW microbenchmark over 8 GiB
and the permutation at 2^30, each under every setting.  One JSON line per
(setting, measurement) on stdout."""
import ctypes as C
import json
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import paper_2103_01216_b200 as pip  # noqa: E402

lib = pip._lib.load()
dev = torch.cuda.current_device()
st = torch.cuda.current_stream().cuda_stream
# the limit belongs to the (primary) context, which libpip's kernels share:
# set it through the CUDA runtime torch loads
import nvidia  # noqa: E402

rt = C.CDLL(str(Path(nvidia.__path__[0]) / "cuda_runtime" / "lib" / "libcudart.so.12"))
LIMIT_L2_FETCH = 0x05  # cudaLimitMaxL2FetchGranularity


def l2_fetch(bytes_=None):
    cur = C.c_size_t(0)
    assert rt.cudaDeviceGetLimit(C.byref(cur), LIMIT_L2_FETCH) == 0
    if bytes_ is not None:
        assert rt.cudaDeviceSetLimit(LIMIT_L2_FETCH, C.c_size_t(bytes_)) == 0
    return cur.value


torch.zeros(1, device="cuda")
prev = C.c_int(l2_fetch())
print(json.dumps({"default_l2_fetch": prev.value}), flush=True)
log2n = int(sys.argv[1]) if len(sys.argv) > 1 else 30
n = 1 << log2n
buf = torch.zeros(n, dtype=torch.int64, device="cuda")
h = torch.empty(n, dtype=torch.int64, device="cuda")
pip.Rng(1).swaps_device(0, n, device=dev, out=h)
a = torch.empty(n, dtype=torch.int64, device="cuda")
prefix = pip.EpsilonConfig(0.5).prefix_words(n)
wb = lib.pip_rp_workspace_bytes(n, prefix, 3)
ws = torch.empty(wb, dtype=torch.uint8, device="cuda")
stats = pip._lib.PipRpStats()
for g in [prev.value, 32, 64, 128, 0, prev.value]:
    l2_fetch(g)
    ms = C.c_float(0)
    lib.pip_bench_random_rmw(buf.data_ptr(), n, n, 7, C.byref(ms), st)
    ts = []
    for _ in range(3):
        a.copy_(torch.arange(n, dtype=torch.int64, device="cuda"))
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        rc = lib.pip_random_permutation_u64(a.data_ptr(), h.data_ptr(), n, prefix, 3, 0, None, 0, None,
                                            ws.data_ptr(), wb, C.byref(stats), st)
        e1.record()
        torch.cuda.synchronize()
        assert rc == 0, rc
        ts.append(e0.elapsed_time(e1))
    print(json.dumps({"l2_fetch": g, "rmw_G_per_s": n / ms.value / 1e6, "rp_ms": ts}), flush=True)
l2_fetch(prev.value)
