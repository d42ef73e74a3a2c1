"""Small invocations of every kernel family, for compute-sanitizer runs."""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np
import torch

import paper_2103_01216_b200 as pip

rng = np.random.default_rng(0)
for n in (1, 7, 8192, 8193, 100_003, 300_000):
    x = rng.integers(0, 1 << 20, size=n, dtype=np.uint64)
    t = torch.from_numpy(x.view(np.int64).copy()).cuda()
    pip.strong.scan_inclusive(t)
    t = torch.from_numpy(x.view(np.int64).copy()).cuda()
    pip.strong.filter_kway(t, pip.pred.mod_eq(3, 0))
    xa = np.sort(x[: n // 2])
    xb = np.sort(x[n // 2:])
    t = torch.from_numpy(np.concatenate([xa, xb]).view(np.int64)).cuda()
    pip.relaxed.merge_relaxed(t, len(xa))
    t2 = torch.from_numpy(np.concatenate([xa, xb]).view(np.int64)).cuda()
    pip.strong.merge_strong(t2, len(xa))
    h = pip.relaxed.make_swap_sequence(n, pip.Rng(3))
    a = torch.arange(n, dtype=torch.int64, device="cuda")
    pip.relaxed.random_permutation(a, torch.from_numpy(h.view(np.int64)).cuda())
    pip.relaxed.random_permutation(a, torch.from_numpy(h.view(np.int64)).cuda(), variant="naive",
                                   budget=pip.EpsilonConfig(0.5, 1e-12))
torch.cuda.synchronize()
print("sanitize smoke ok")
