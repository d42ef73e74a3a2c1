"""Timings of the SURVEY §8(f) rows beyond the BASELINE configs (one JSON
line each): list ranking / contraction (rows 4) and quicksort (row 3), CUDA
events around the call on device-resident inputs, setup untimed.

usage: python tools/bench_extra.py [--log2n 24] [--reps 3] [--only list|quicksort]
"""
import argparse
import json
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))

import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2103_01216_b200 as pip  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--log2n", type=int, default=24)
ap.add_argument("--reps", type=int, default=3)
ap.add_argument("--only", choices=["list", "quicksort", "tree"], default=None)
args = ap.parse_args()
n = 1 << args.log2n
dev = "cuda:0"
NIL = -1  # all-ones as int64


def timed(setup, body):
    ts = []
    for _ in range(args.reps + 1):
        st = setup()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        t0 = time.perf_counter()
        e0.record()
        out = body(st)
        e1.record()
        e1.synchronize()
        ts.append((e0.elapsed_time(e1), time.perf_counter() - t0, out))
    return ts[1:]


if args.only in (None, "list"):
    # one random chain over n elements (order = a GPU random permutation)
    order = torch.arange(n, dtype=torch.int64, device=dev)
    h = pip.Rng(1).swaps_device(0, n)
    pip.relaxed.random_permutation(order, h)
    p = torch.arange(n, dtype=torch.int64, device=dev)
    pip.relaxed.random_permutation(p, pip.Rng(2).swaps_device(0, n))


    def chain():
        nxt = torch.full((n,), NIL, dtype=torch.int64, device=dev)
        prv = torch.full((n,), NIL, dtype=torch.int64, device=dev)
        nxt[order[:-1]] = order[1:]
        prv[order[1:]] = order[:-1]
        return pip.contraction.LinkedList(nxt, prv)


    budget = pip.EpsilonConfig(0.5)
    for name in ("list_rank", "list_contract"):
        fn = pip.contraction.list_rank if name == "list_rank" else pip.contraction.list_contract
        res = timed(chain, lambda l, fn=fn: fn(l, p, budget=budget))
        ms = sorted(r[0] for r in res)[len(res) // 2]
        line = {"op": name, "n": n, "ms": ms, "elements_per_s": n / (ms / 1e3),
                "rounds": None, "budget": "EpsilonConfig(0.5) (f=0.02)",
                "note": "host-driven rounds (one sync per round) + in-place rank waves; single chain, "
                        "random order and priorities from the GPU permutation"}
        if name == "list_contract":
            line["rounds"] = res[-1][2].rounds
        if name == "list_rank":
            lst = chain()
            r = pip.contraction.list_rank(lst, p, budget=budget)
            ref = torch.empty(n, dtype=torch.int64, device=dev)
            ref[order] = torch.arange(n, dtype=torch.int64, device=dev)
            line["verified"] = bool(torch.equal(r, ref))
        print(json.dumps(line), flush=True)

if args.only in (None, "tree"):
    # a complete binary tree of n - 1 nodes with randomly permuted ids (node
    # k has children 2k+1, 2k+2), random priorities and values; the folded
    # value of the single root must be the sum of all values mod 2^64
    m = n - 1
    perm = torch.arange(m, dtype=torch.int64, device=dev)
    pip.relaxed.random_permutation(perm, pip.Rng(7).swaps_device(0, m))
    k = torch.arange(m, dtype=torch.int64, device=dev)
    internal = k < (m - 1) // 2
    pa0 = torch.full((m,), NIL, dtype=torch.int64, device=dev)
    lf0 = torch.full((m,), NIL, dtype=torch.int64, device=dev)
    rt0 = torch.full((m,), NIL, dtype=torch.int64, device=dev)
    ki = k[internal]
    lf0[perm[ki]] = perm[2 * ki + 1]
    rt0[perm[ki]] = perm[2 * ki + 2]
    pa0[perm[2 * ki + 1]] = perm[ki]
    pa0[perm[2 * ki + 2]] = perm[ki]
    pt = torch.arange(m, dtype=torch.int64, device=dev)
    pip.relaxed.random_permutation(pt, pip.Rng(8).swaps_device(0, m))
    v0 = pip.Rng(9).words_device(0, m)
    want = int(v0.cpu().numpy().view(np.uint64).sum(dtype=np.uint64))

    def tree_setup():
        return (pip.contraction.BinaryTree(pa0.clone(), lf0.clone(), rt0.clone()), v0.clone())

    res = timed(tree_setup, lambda st: pip.contraction.tree_contract(st[0], pt, st[1]))
    ms = sorted(r[0] for r in res)[len(res) // 2]
    roots, stats = res[-1][2]
    print(json.dumps({"op": "tree_contract", "n": m, "ms": ms, "elements_per_s": m / (ms / 1e3),
                      "rounds": stats.rounds, "budget": "EpsilonConfig(0.5) (f=0.02)",
                      "verified": roots == {int(perm[0].item()): want},
                      "note": "round loop on the device (csrc/tree.cu): frontier ring, sweep, "
                              "active set and rake-parent map in device memory; the host reads a "
                              "few counts per round.  Complete binary tree, random ids"}),
          flush=True)

if args.only in (None, "quicksort"):
    x0 = pip.Rng(3).words_device(0, n)
    res = timed(lambda: x0.clone(), lambda t: pip.strong.quicksort_strong(t, pip.Rng(5)))
    ms = sorted(r[0] for r in res)[len(res) // 2]
    t = x0.clone()
    pip.strong.quicksort_strong(t, pip.Rng(5))
    u = t.cpu().numpy().view(np.uint64)
    print(json.dumps({"op": "quicksort_strong", "n": n, "ms": ms, "elements_per_s": n / (ms / 1e3),
                      "verified": bool(np.all(u[1:] >= u[:-1])),
                      "note": "level-batched host recursion over the GPU partition (3 syncs per level) + "
                              "one grid-wide bitonic network for the <= 2^22-word leaves"}),
          flush=True)
