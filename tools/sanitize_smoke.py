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
# round 2 entry points: reservation table, compaction, move, tree contraction
from paper_2103_01216_b200 import detres, runtime  # noqa: E402

t = detres.ReservationTable(1 << 12)
k = torch.arange(0, 3000, 3, dtype=torch.int64, device="cuda")
t.reserve_max(k, k * 2)
t.lookup(k)
t.delete(k[::2])
for n in (1, 1000, 100_003):
    x = rng.integers(0, 1 << 63, size=n, dtype=np.uint64)
    d = torch.from_numpy(x.view(np.int64).copy()).cuda()
    runtime.compact_by_mask(d, torch.from_numpy(rng.random(n) < 0.5).cuda(), n)
    pip.relaxed.filter_relaxed(d, pip.pred.even(), pip.EpsilonConfig(0.5, 0.05))
    pip.relaxed.partition_relaxed(d, pip.pred.even(), pip.EpsilonConfig(0.5, 0.05))
m = 2 ** 12 - 1
perm = np.random.default_rng(1).permutation(m)
NILW = np.uint64(2 ** 64 - 1)
pa = np.full(m, NILW, dtype=np.uint64)
lf = np.full(m, NILW, dtype=np.uint64)
rt = np.full(m, NILW, dtype=np.uint64)
for q in range((m - 1) // 2):
    lf[perm[q]], rt[perm[q]] = perm[2 * q + 1], perm[2 * q + 2]
    pa[perm[2 * q + 1]] = pa[perm[2 * q + 2]] = perm[q]
tree = pip.contraction.BinaryTree(pa, lf, rt)
pip.contraction.tree_contract(tree, pip.contraction.make_priorities(m, pip.Rng(2)),
                              np.ones(m, dtype=np.uint64))
torch.cuda.synchronize()
print("sanitize smoke ok")
