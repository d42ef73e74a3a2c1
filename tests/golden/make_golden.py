"""Generate the golden fixtures from the reference `pipal` itself.

Run in the build container (the reference is importable there, not on the
GPU box):  PYTHONPATH=/root/reference/pkg/src python tests/golden/make_golden.py

Every fixture is produced by calling the reference's own public functions on
seeded inputs (the same seeds its tests use where they have one), so the GPU
parity tests compare against the reference's outputs, not a restatement.
"""
from __future__ import annotations

import sys
from pathlib import Path

import numpy as np

sys.dont_write_bytecode = True
sys.path.insert(0, "/root/reference/pkg/src")

from pipal import baselines as bl  # noqa: E402
from pipal import relaxed, strong  # noqa: E402
from pipal.runtime import EpsilonConfig, Rng, WORD  # noqa: E402

OUT = Path(__file__).resolve().parent


def rand_words(seed, n, hi=None):
    rng = np.random.default_rng(seed)
    if hi is None:
        return rng.integers(0, 1 << 64, size=n, dtype=np.uint64)
    return rng.integers(0, hi, size=n, dtype=np.uint64)


def make_scan():
    d = {}
    cases = {
        "one": np.array([7], dtype=np.uint64),
        "ones": np.array([1, 1, 1, 1], dtype=np.uint64),
        "pi": np.array([3, 1, 4, 1, 5, 9, 2, 6], dtype=np.uint64),
        "wrap": np.array([(1 << 64) - 1, 5], dtype=np.uint64),
    }
    for n in [2, 3, 255, 256, 257, 1000, 4096, 12345]:  # test_strong.py:96-101
        cases[f"rand{n}"] = rand_words(n, n)
    cases["c1like"] = Rng(1).words(0, 70_000) >> WORD(44)  # BASELINE config 1 values
    for name, x in cases.items():
        a = x.copy()
        r = strong.scan(a)  # the reference's in-place Alg. 3
        d["in_" + name] = x
        d["out_" + name] = a
        d["tot_" + name] = np.array([r.total], dtype=np.uint64)
    np.savez_compressed(OUT / "scan.npz", **d)


def make_filter():
    d = {}
    preds = {
        "even": lambda b: (b & WORD(1)) == 0,        # cli.py:41
        "odd": lambda b: (b & WORD(1)) == 1,         # test_strong.py:184
        "mod3": lambda b: (b % WORD(3)) == 0,        # BASELINE config 2
    }
    inputs = {str(n): rand_words(n + 17, n) for n in [0, 1, 10, 1000, 9999, 20000]}
    inputs["c2like"] = Rng(1).words(0, 20_000) >> WORD(1)  # config 2 value distribution
    for name, x in inputs.items():
        d[f"in_{name}"] = x
        for pname, p in preds.items():
            a = x.copy()
            m = strong.filter_kway(a, p)  # test_strong.py:170-176
            d[f"out_{pname}_{name}"] = a[:m].copy()
    np.savez_compressed(OUT / "filter.npz", **d)


def make_partition():
    d = {}
    preds = {
        "even": lambda b: (b & WORD(1)) == 0,        # test_strong.py:204
        "mod3": lambda b: (b % WORD(3)) == 0,        # the config-2 predicate
        "le2e62": lambda b: b <= WORD(1 << 62),      # pivot-style (quicksort_strong)
    }
    inputs = {str(n): rand_words(n + 3, n) for n in [0, 1, 17, 1000, 30_000]}  # test_strong.py:200
    for name, x in inputs.items():
        d[f"in_{name}"] = x
        for pname, p in preds.items():
            a = x.copy()
            m = strong.partition_unstable(a, p)
            d[f"out_{pname}_{name}"] = a
            d[f"m_{pname}_{name}"] = np.array([m], dtype=np.uint64)
    np.savez_compressed(OUT / "partition.npz", **d)


def make_contraction():
    from pipal.contraction import LinkedList, list_contract, list_rank, make_priorities
    from pipal.runtime import NIL, POWER_ONLY_FRACTION

    def random_chains(rng, n, nchains):  # test_contraction.py:45-59
        order = rng.permutation(n)
        cuts = np.sort(rng.choice(np.arange(1, n), size=nchains - 1, replace=False)) \
            if nchains > 1 else np.array([], dtype=np.int64)
        nxt = np.full(n, NIL, dtype=np.uint64)
        prv = np.full(n, NIL, dtype=np.uint64)
        prev_cut = 0
        for cut in list(cuts) + [n]:
            seg = order[prev_cut:cut]
            for a, b in zip(seg, seg[1:]):
                nxt[a] = b
                prv[b] = a
            prev_cut = cut
        return nxt, prv

    d = {}
    cases = [("c1", 1, 1, 0.5, 1.0), ("c9", 9, 1, 0.5, 1.0), ("c4000", 4000, 7, 0.5, 0.02),
             ("c2000p3", 2000, 40, 0.3, POWER_ONLY_FRACTION),
             ("c50000", 50_000, 3, 0.5, POWER_ONLY_FRACTION)]
    for name, n, nch, eps, frac in cases:
        rng = np.random.default_rng(n + nch)
        nxt, prv = random_chains(rng, n, nch)
        p = make_priorities(n, Rng(n))
        budget = EpsilonConfig(eps, prefix_fraction=frac)
        d[f"next_{name}"], d[f"prev_{name}"], d[f"p_{name}"] = nxt.copy(), prv.copy(), p.copy()
        d[f"budget_{name}"] = np.array([eps, frac])
        lst = LinkedList(nxt.copy(), prv.copy())
        trace = []
        st = list_contract(lst, p, budget=budget, trace=trace)
        d[f"cnext_{name}"], d[f"cprev_{name}"] = lst.next, lst.prev
        d[f"ccounts_{name}"] = np.array(st.committed_per_round, dtype=np.uint64)
        d[f"ctrace_{name}"] = np.concatenate(trace) if trace else np.zeros(0, dtype=np.uint64)
        lst = LinkedList(nxt.copy(), prv.copy())
        sink = []
        ranks = list_rank(lst, p, budget=budget, stats_sink=sink)
        d[f"ranks_{name}"] = ranks.copy()
        d[f"rcounts_{name}"] = np.array(sink[0].committed_per_round, dtype=np.uint64)
    # tree contraction (contraction.py:528-559): random full binary trees
    from pipal.contraction import BinaryTree, tree_contract

    def random_full_binary_tree(rng, n):  # test_contraction.py:63-83
        ids = rng.permutation(n)
        parent = np.full(n, NIL, dtype=np.uint64)
        left = np.full(n, NIL, dtype=np.uint64)
        right = np.full(n, NIL, dtype=np.uint64)
        leaves = [int(ids[0])]
        used = 1
        while used < n:
            pick = int(rng.integers(0, len(leaves)))
            node = leaves.pop(pick)
            l, r = int(ids[used]), int(ids[used + 1])
            used += 2
            left[node] = l
            right[node] = r
            parent[l] = node
            parent[r] = node
            leaves.extend([l, r])
        return parent, left, right

    tcases = [("t1", 1, 0.5, 1.0), ("t3", 3, 0.5, 1.0), ("t999", 999, 0.3, POWER_ONLY_FRACTION),
              ("t5001", 5001, 0.5, POWER_ONLY_FRACTION), ("t20001", 20001, 0.5, 0.02)]
    for name, n, eps, frac in tcases:
        rng = np.random.default_rng(n)
        pa, lf, rt = random_full_binary_tree(rng, n)
        vals = rng.integers(0, 1 << 64, size=n, dtype=np.uint64)
        p = make_priorities(n, Rng(n + 1))
        budget = EpsilonConfig(eps, prefix_fraction=frac)
        d[f"tpa_{name}"], d[f"tlf_{name}"], d[f"trt_{name}"] = pa.copy(), lf.copy(), rt.copy()
        d[f"tval_{name}"], d[f"tp_{name}"] = vals.copy(), p.copy()
        d[f"tbudget_{name}"] = np.array([eps, frac])
        t = BinaryTree(pa, lf, rt)
        v = vals.copy()
        trace = []
        roots, st = tree_contract(t, p, v, budget=budget, trace=trace, debug=True)
        d[f"troots_{name}"] = np.array(sorted(roots.items()), dtype=np.uint64).reshape(-1, 2)
        d[f"tcounts_{name}"] = np.array(st.committed_per_round, dtype=np.uint64)
        d[f"ttrace_{name}"] = np.concatenate(trace) if trace else np.zeros(0, dtype=np.uint64)
        d[f"tvout_{name}"] = v
        d[f"tpaout_{name}"], d[f"tlfout_{name}"], d[f"trtout_{name}"] = t.parent, t.left, t.right
    np.savez_compressed(OUT / "contraction.npz", **d)


def make_merge():
    d = {}
    pairs = [(1, 1), (5, 3), (100, 1), (1, 100), (1000, 1000), (4096, 999)]  # test_strong.py:248
    for na, nb in pairs:
        rng = np.random.default_rng(na * 7919 + nb)
        x = np.sort(rng.integers(0, 50, size=na, dtype=np.uint64))
        y = np.sort(rng.integers(0, 50, size=nb, dtype=np.uint64))
        a = np.concatenate([x, y])
        strong.merge_strong(a, na)
        d[f"in_small{na}_{nb}"] = np.concatenate([x, y])
        d[f"split_small{na}_{nb}"] = np.array([na], dtype=np.uint64)
        d[f"out_small{na}_{nb}"] = a
    for na, nb, eps in [(10_000, 3777, 0.5), (999, 65_536, 0.3), (20_000, 20_000, 0.7)]:
        rng = np.random.default_rng(na * 131 + nb)  # test_relaxed_seq.py:36-40
        x = np.sort(rng.integers(0, 2000, size=na, dtype=np.uint64))
        y = np.sort(rng.integers(0, 2000, size=nb, dtype=np.uint64))
        a = np.concatenate([x, y])
        relaxed.merge_relaxed(a, na, EpsilonConfig(eps, 1e-12))
        d[f"in_relaxed{na}_{nb}"] = np.concatenate([x, y])
        d[f"split_relaxed{na}_{nb}"] = np.array([na], dtype=np.uint64)
        d[f"out_relaxed{na}_{nb}"] = a
    # config-3-like: heavy duplicates, values < 2^30
    x = np.sort(Rng(1).words(0, 40_000) >> WORD(34))
    y = np.sort(Rng(2).words(0, 40_000) >> WORD(34))
    a = np.concatenate([x, y])
    strong.merge_strong(a, len(x))
    d["in_c3like"] = np.concatenate([x, y])
    d["split_c3like"] = np.array([len(x)], dtype=np.uint64)
    d["out_c3like"] = a
    np.savez_compressed(OUT / "merge.npz", **d)


def make_rp():
    d = {}
    cases = [
        ("fig3", np.array([0, 0, 1, 3, 1, 2, 3, 1], dtype=np.uint64), 0.5, 1.0),
        ("n10000_s177", relaxed.make_swap_sequence(10_000, Rng(177)), 0.5, 0.02),
        ("n3000_s9", relaxed.make_swap_sequence(3000, Rng(9)), 0.5, 0.02),
        ("n5000_s21", relaxed.make_swap_sequence(5000, Rng(21)), 0.5, 0.02),
        ("n4001_pure03", relaxed.make_swap_sequence(4001, Rng(4)), 0.3, 1e-12),
        ("n20000_pure07", relaxed.make_swap_sequence(20_000, Rng(3)), 0.7, 1e-12),
    ]
    for name, h, eps, frac in cases:
        for variant in relaxed.RP_VARIANTS:
            n = len(h)
            a = np.arange(n, dtype=np.uint64)
            tr = []
            st = relaxed.random_permutation(a, h, variant, EpsilonConfig(eps, frac), trace=tr)
            ref = np.arange(n, dtype=np.uint64)
            bl.seq_knuth_shuffle(ref, h)
            assert np.array_equal(a, ref)
            key = f"{name}_{variant}"
            d[key + "__h"] = h
            d[key + "__budget"] = np.array([eps, frac], dtype=np.float64)
            d[key + "__variant"] = np.array([variant])
            d[key + "__rounds"] = np.array([st.rounds], dtype=np.uint64)
            d[key + "__committed"] = np.array(st.committed_per_round, dtype=np.uint64)
            d[key + "__peak"] = np.array([st.peak_table_load], dtype=np.float64)
            d[key + "__trace"] = (np.concatenate(tr) if tr else np.empty(0, np.uint64)).astype(np.uint64)
            d[key + "__out"] = a
    np.savez_compressed(OUT / "rp.npz", **d)


def make_rng():
    d = {}
    for seed in (0, 1, 177, (1 << 64) - 1):
        r = Rng(seed)
        d[f"words_{seed}"] = r.words(5, 5000)
        d[f"swaps_{seed}"] = relaxed.make_swap_sequence(3000, r)
    np.savez_compressed(OUT / "rng.npz", **d)


def make_tree_ops():
    """Tree contraction on a forest (three random full binary trees with
    interleaved ids, plus a bare node) under every combine the device folds
    with (np.add / maximum / minimum / bitwise_xor): rounds, traces, roots,
    folded values and the final forest from the reference itself."""
    from pipal.contraction import BinaryTree, make_priorities, tree_contract
    from pipal.runtime import NIL, POWER_ONLY_FRACTION

    rng = np.random.default_rng(77)
    sizes = [301, 1, 77, 1023]
    n = sum(sizes)
    ids = rng.permutation(n)
    pa = np.full(n, NIL, dtype=np.uint64)
    lf = np.full(n, NIL, dtype=np.uint64)
    rt = np.full(n, NIL, dtype=np.uint64)
    base = 0
    for sz in sizes:
        mine = ids[base:base + sz]
        base += sz
        leaves = [int(mine[0])]
        used = 1
        while used < sz:
            node = leaves.pop(int(rng.integers(0, len(leaves))))
            l, r = int(mine[used]), int(mine[used + 1])
            used += 2
            lf[node], rt[node] = l, r
            pa[l] = pa[r] = node
            leaves.extend([l, r])
    vals = rng.integers(0, 1 << 64, size=n, dtype=np.uint64)
    p = make_priorities(n, Rng(5))
    d = {"pa": pa, "lf": lf, "rt": rt, "vals": vals, "p": p}
    for cname, comb in (("add", np.add), ("max", np.maximum), ("min", np.minimum),
                        ("xor", np.bitwise_xor)):
        t = BinaryTree(pa.copy(), lf.copy(), rt.copy())
        v = vals.copy()
        trace = []
        roots, st = tree_contract(t, p, v, budget=EpsilonConfig(0.5, POWER_ONLY_FRACTION),
                                  combine=comb, trace=trace, debug=True)
        d[f"roots_{cname}"] = np.array(sorted(roots.items()), dtype=np.uint64).reshape(-1, 2)
        d[f"counts_{cname}"] = np.array(st.committed_per_round, dtype=np.uint64)
        d[f"trace_{cname}"] = np.concatenate(trace)
        d[f"vout_{cname}"] = v
        d[f"paout_{cname}"], d[f"lfout_{cname}"], d[f"rtout_{cname}"] = t.parent, t.left, t.right
    np.savez_compressed(OUT / "tree_ops.npz", **d)


def make_detres():
    """ReservationTable slot layouts after seeded batches (detres.py:40-211):
    the device table reproduces the reference's probe steps, so its key and
    value arrays must equal these word for word; plus compact_by_mask."""
    from pipal import detres
    from pipal.runtime import compact_by_mask

    d = {}
    cases = {
        "small": (16, [(np.array([5, 5, 5], dtype=np.uint64), np.array([3, 9, 5], dtype=np.uint64))]),
        "collide": (32, [(np.array([1, 9, 17, 25, 33], dtype=np.uint64),) * 2]),
    }
    rng = np.random.default_rng(42)
    keys = rng.integers(0, 500, size=10_000, dtype=np.uint64)
    vals = rng.integers(0, 1 << 63, size=10_000, dtype=np.uint64)
    cases["batches"] = (2048, [(keys[s:s + 700], vals[s:s + 700]) for s in range(0, 10_000, 700)])
    big_k = rng.integers(0, 1 << 64, size=7_000, dtype=np.uint64)
    big_v = rng.integers(0, 1 << 64, size=7_000, dtype=np.uint64)
    cases["dense"] = (1 << 14, [(big_k[:5_000], big_v[:5_000]), (big_k[3_000:], big_v[3_000:])])
    for name, (cap, batches) in cases.items():
        t = detres.ReservationTable(cap)
        for i, (k, v) in enumerate(batches):
            d[f"{name}_k{i}"] = k
            d[f"{name}_v{i}"] = v
            t.reserve_max(k, v)
        d[f"{name}_cap"] = np.array([cap, len(batches), t.count], dtype=np.uint64)
        d[f"{name}_peak"] = np.array([t.peak_load])
        d[f"{name}_keys"] = t.keys.copy()
        d[f"{name}_vals"] = np.where(t.keys != np.uint64((1 << 64) - 1), t.vals, 0).astype(np.uint64)
        dk = batches[0][0][::2]
        t.delete(dk)
        d[f"{name}_delk"] = dk
        d[f"{name}_keys_after_delete"] = t.keys.copy()
        d[f"{name}_count_after_delete"] = np.array([t.count], dtype=np.uint64)
    for n in (1, 255, 256, 257, 10_000, 20_011):
        a = rand_words(n + 1, n)
        keep = np.random.default_rng(n).random(n) < 0.37
        b = a.copy()
        m = compact_by_mask(b, keep, n)
        d[f"compact_in_{n}"] = a
        d[f"compact_keep_{n}"] = keep
        d[f"compact_out_{n}"] = b[:m]
    np.savez_compressed(OUT / "detres.npz", **d)


if __name__ == "__main__":
    make_tree_ops()
    make_detres()
    make_scan()
    make_filter()
    make_partition()
    make_contraction()
    make_merge()
    make_rp()
    make_rng()
    for p in sorted(OUT.glob("*.npz")):
        print(p.name, p.stat().st_size)
