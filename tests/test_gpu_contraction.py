"""GPU parity: list contraction and list ranking (contraction.py:264-365)
against the reference's own outputs (tests/golden/contraction.npz, made by
tests/golden/make_golden.py): identical final slots, ranks, RoundStats and
per-round committed sets; plus the reference's known answers
(test_contraction.py:110-210)."""
from __future__ import annotations

import numpy as np
import pytest

from conftest import golden

pytestmark = pytest.mark.gpu

NIL = (1 << 64) - 1


@pytest.fixture(scope="module")
def pip():
    import paper_2103_01216_b200 as pip

    return pip


def words(vals):
    return np.array([NIL if v is None else v for v in vals], dtype=np.uint64)


def chain_list(pip, order):
    n = len(order)
    nxt = np.full(n, NIL, dtype=np.uint64)
    prv = np.full(n, NIL, dtype=np.uint64)
    for a, b in zip(order, order[1:]):
        nxt[a] = b
        prv[b] = a
    return pip.contraction.LinkedList(nxt, prv)


def seq_list_rank(nxt, prv):  # baselines.py:57-72
    n = len(nxt)
    ranks = np.zeros(n, dtype=np.uint64)
    for head in np.flatnonzero(prv == np.uint64(NIL)):
        r, v = 0, int(head)
        while v != NIL:
            ranks[v] = r
            r += 1
            v = int(nxt[v])
    return ranks


CASES = ["c1", "c9", "c4000", "c2000p3", "c50000"]


@pytest.mark.parametrize("name", CASES)
@pytest.mark.parametrize("where", ["host", "device"])
def test_list_contract_golden(pip, name, where):
    import torch

    g = golden("contraction")
    eps, frac = g[f"budget_{name}"]
    budget = pip.EpsilonConfig(float(eps), float(frac))
    nxt, prv, p = g[f"next_{name}"].copy(), g[f"prev_{name}"].copy(), g[f"p_{name}"]
    if where == "device":
        lst = pip.contraction.LinkedList(torch.from_numpy(nxt.view(np.int64)).cuda(),
                                         torch.from_numpy(prv.view(np.int64)).cuda())
    else:
        lst = pip.contraction.LinkedList(nxt, prv)
    trace: list = []
    st = pip.contraction.list_contract(lst, p, budget=budget, trace=trace)
    out_n = lst.next if where == "host" else lst.next.cpu().numpy().view(np.uint64)
    out_p = lst.prev if where == "host" else lst.prev.cpu().numpy().view(np.uint64)
    assert np.array_equal(out_n, g[f"cnext_{name}"]) and np.array_equal(out_p, g[f"cprev_{name}"])
    assert st.committed_per_round == g[f"ccounts_{name}"].tolist()
    assert st.rounds == len(g[f"ccounts_{name}"])
    assert np.array_equal(np.concatenate(trace), g[f"ctrace_{name}"])


@pytest.mark.parametrize("name", CASES)
def test_list_rank_golden(pip, name):
    g = golden("contraction")
    eps, frac = g[f"budget_{name}"]
    budget = pip.EpsilonConfig(float(eps), float(frac))
    lst = pip.contraction.LinkedList(g[f"next_{name}"].copy(), g[f"prev_{name}"].copy())
    sink: list = []
    ranks = pip.contraction.list_rank(lst, g[f"p_{name}"], budget=budget, stats_sink=sink)
    assert np.array_equal(ranks, g[f"ranks_{name}"])
    assert np.array_equal(ranks, seq_list_rank(g[f"next_{name}"], g[f"prev_{name}"]))
    assert sink[0].committed_per_round == g[f"rcounts_{name}"].tolist()


def test_make_priorities_matches_reference(pip):
    g = golden("contraction")
    for name in CASES:
        n = len(g[f"p_{name}"])
        assert np.array_equal(pip.contraction.make_priorities(n, pip.Rng(n)), g[f"p_{name}"])


def test_known_answers(pip):
    FULL = pip.EpsilonConfig(0.5, 1.0)
    C = pip.contraction
    # test_contraction.py:110-113
    st = C.list_contract(C.LinkedList(words([None]), words([None])), words([0]), budget=FULL)
    assert st.rounds == 1 and st.committed_per_round == [1]
    # :116-128 worked instance: first round contracts priorities {1,2,3,4}; 4 rounds
    lst = chain_list(pip, list(range(9)))
    p = words([v - 1 for v in [5, 1, 6, 2, 9, 3, 7, 4, 8]])
    trace: list = []
    st = C.list_contract(lst, p, budget=FULL, trace=trace)
    assert sorted((p[trace[0]] + np.uint64(1)).tolist()) == [1, 2, 3, 4]
    assert st.rounds == 4 and st.total_committed == 9
    # :131-147 splice-time context
    lst = chain_list(pip, [3, 1, 4, 0, 2])
    observed = {}

    def on_splice(v, u, x):
        for vi, ui, xi in zip(v.tolist(), u.tolist(), x.tolist()):
            observed[vi] = (ui, xi)

    C.list_contract(lst, words([4, 0, 3, 2, 1]), on_splice=on_splice, budget=FULL)
    assert observed[1] == (3, 4) and set(observed) == {0, 1, 2, 3, 4}
    for v, (u, x) in observed.items():
        assert lst.prev[v] == u and lst.next[v] == x
    # :161-169 ranks
    assert C.list_rank(C.LinkedList(words([None]), words([None])), words([0]), budget=FULL).tolist() == [0]
    assert C.list_rank(chain_list(pip, [0, 1, 2]), words([2, 0, 1]), budget=FULL).tolist() == [0, 1, 2]


def test_validate_rejects(pip):
    C = pip.contraction
    with pytest.raises(ValueError):
        C.validate_linked_list(C.LinkedList(words([1, None]), words([None, None])))
    with pytest.raises(ValueError, match="cycle"):
        C.validate_linked_list(C.LinkedList(words([1, 0]), words([1, 0])))


def test_rank_budget_metered_large(pip):
    # test_contraction.py:193-210 at a larger size: charged <= 8 b, ranks exact
    rng = np.random.default_rng(8)
    n = 400_000
    order = rng.permutation(n)
    nxt = np.full(n, NIL, dtype=np.uint64)
    prv = np.full(n, NIL, dtype=np.uint64)
    nxt[order[:-1]] = order[1:]
    prv[order[1:]] = order[:-1]
    ref = np.empty(n, dtype=np.uint64)
    ref[order] = np.arange(n, dtype=np.uint64)
    p = pip.contraction.make_priorities(n, pip.Rng(10))
    cfg = pip.EpsilonConfig(0.5, 1e-12)
    b = cfg.prefix_words(n)
    meter = pip.SpaceMeter()
    out = {}
    rep = pip.meter_scope(meter, 8 * b, lambda: out.__setitem__(
        "r", pip.contraction.list_rank(pip.contraction.LinkedList(nxt, prv), p, cfg)))
    assert rep.peak_words <= 8 * b and meter.current_words == 0
    assert np.array_equal(out["r"], ref)


# ----------------------------------------------------------------- trees

TCASES = ["t1", "t3", "t999", "t5001", "t20001"]


@pytest.mark.parametrize("name", TCASES)
@pytest.mark.parametrize("where", ["host", "device"])
def test_tree_contract_golden(pip, name, where):
    import torch

    g = golden("contraction")
    eps, frac = g[f"tbudget_{name}"]
    budget = pip.EpsilonConfig(float(eps), float(frac))
    arrs = [g[f"tpa_{name}"].copy(), g[f"tlf_{name}"].copy(), g[f"trt_{name}"].copy()]
    vals = g[f"tval_{name}"].copy()
    if where == "device":
        arrs = [torch.from_numpy(x.view(np.int64)).cuda() for x in arrs]
        vals = torch.from_numpy(vals.view(np.int64)).cuda()
    tree = pip.contraction.BinaryTree(*arrs)
    trace: list = []
    roots, st = pip.contraction.tree_contract(tree, g[f"tp_{name}"], vals, budget=budget,
                                              trace=trace, debug=True)
    want = {int(a): int(b) for a, b in g[f"troots_{name}"].tolist()}
    assert roots == want
    assert st.committed_per_round == g[f"tcounts_{name}"].tolist()
    assert np.array_equal(np.concatenate(trace), g[f"ttrace_{name}"])

    def h(x):
        return x if isinstance(x, np.ndarray) else x.cpu().numpy().view(np.uint64)

    assert np.array_equal(h(vals), g[f"tvout_{name}"])
    for arr, key in zip((tree.parent, tree.left, tree.right), ("tpaout", "tlfout", "trtout")):
        assert np.array_equal(h(arr), g[f"{key}_{name}"])


def test_tree_known_answers(pip):
    C = pip.contraction
    FULL = pip.EpsilonConfig(0.5, 1.0)
    # test_contraction.py:213-246
    t = C.BinaryTree(words([None]), words([None]), words([None]))
    roots, st = C.tree_contract(t, words([0]), words([42]), budget=FULL)
    assert roots == {0: 42} and st.rounds == 1
    t = C.BinaryTree(words([None, 0, 0]), words([1, None, None]), words([2, None, None]))
    roots, _ = C.tree_contract(t, words([2, 0, 1]), words([10, 20, 30]), budget=FULL, debug=True)
    assert roots == {0: 60}
    t = C.BinaryTree(words([None, None, None]), words([None] * 3), words([None] * 3))
    roots, _ = C.tree_contract(t, words([2, 0, 1]), words([5, 6, 7]), budget=FULL)
    assert roots == {0: 5, 1: 6, 2: 7}
    with pytest.raises(ValueError, match="exactly two children"):
        C.validate_binary_tree(C.BinaryTree(words([None, 0]), words([1, None]), words([None, None])))


def _random_full_binary_tree(rng, n):  # test_contraction.py:63-83
    ids = rng.permutation(n)
    parent = np.full(n, NIL, dtype=np.uint64)
    left = np.full(n, NIL, dtype=np.uint64)
    right = np.full(n, NIL, dtype=np.uint64)
    leaves = [int(ids[0])]
    used = 1
    while used < n:
        node = leaves.pop(int(rng.integers(0, len(leaves))))
        lc, rc = int(ids[used]), int(ids[used + 1])
        used += 2
        left[node], right[node] = lc, rc
        parent[lc] = parent[rc] = node
        leaves.extend([lc, rc])
    return parent, left, right


def _seq_tree_eval(parent, left, right, values):  # baselines.py:75-96
    out = {}
    for root in np.flatnonzero(parent == np.uint64(NIL)).tolist():
        total, stack = 0, [root]
        while stack:
            v = stack.pop()
            total = (total + int(values[v])) & NIL
            for c in (left[v], right[v]):
                if c != np.uint64(NIL):
                    stack.append(int(c))
        out[root] = total
    return out


def test_tree_budget_metered(pip):
    # test_contraction.py:249-265: n = 50_001, pure budget, charged <= 8 b
    rng = np.random.default_rng(3)
    n = 50_001
    pa, lf, rt = _random_full_binary_tree(rng, n)
    vals = rng.integers(0, 1 << 64, size=n, dtype=np.uint64)
    ref = _seq_tree_eval(pa, lf, rt, vals)
    cfg = pip.EpsilonConfig(0.5, 1e-12)
    b = cfg.prefix_words(n)
    p = pip.contraction.make_priorities(n, pip.Rng(2))
    meter = pip.SpaceMeter()
    out = {}
    tree = pip.contraction.BinaryTree(pa, lf, rt)
    rep = pip.meter_scope(meter, 8 * b, lambda: out.__setitem__("r", pip.contraction.tree_contract(
        tree, p, vals, cfg, debug=True)))
    assert rep.peak_words <= 8 * b and meter.current_words == 0
    assert out["r"][0] == ref


@pytest.mark.parametrize("cname", ["add", "max", "min", "xor"])
@pytest.mark.parametrize("where", ["host", "device"])
def test_tree_contract_forest_combine_ops_golden(pip, cname, where):
    """A forest of four trees (one a bare node) under every combine the
    device folds with: the reference's own rounds, traces, roots, folded
    values and final forest (tests/golden/tree_ops.npz)."""
    import torch

    g = golden("tree_ops")
    comb = {"add": np.add, "max": np.maximum, "min": np.minimum, "xor": np.bitwise_xor}[cname]
    arrs = [g["pa"].copy(), g["lf"].copy(), g["rt"].copy()]
    vals = g["vals"].copy()
    if where == "device":
        arrs = [torch.from_numpy(x.view(np.int64)).cuda() for x in arrs]
        vals = torch.from_numpy(vals.view(np.int64)).cuda()
    tree = pip.contraction.BinaryTree(*arrs)
    trace: list = []
    roots, st = pip.contraction.tree_contract(tree, g["p"], vals,
                                              budget=pip.EpsilonConfig(0.5, 1e-12), combine=comb,
                                              trace=trace, debug=True)

    def h(x):
        return x if isinstance(x, np.ndarray) else x.cpu().numpy().view(np.uint64)

    assert roots == {int(a): int(b) for a, b in g[f"roots_{cname}"].tolist()}
    assert st.committed_per_round == g[f"counts_{cname}"].tolist()
    assert np.array_equal(np.concatenate(trace), g[f"trace_{cname}"])
    assert np.array_equal(h(vals), g[f"vout_{cname}"])
    for arr, key in zip((tree.parent, tree.left, tree.right), ("paout", "lfout", "rtout")):
        assert np.array_equal(h(arr), g[f"{key}_{cname}"])
