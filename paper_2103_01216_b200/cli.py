"""Benchmark / verification harness for the GPU path.

Mirrors the reference's ``pipal`` command line (``cli.py:159-394`` registry,
``:396-435`` run_bench, ``:442-614`` parser and subcommands) for the
algorithms on this path, with the same subcommands, exit codes and report
schema so that GPU rows land in the same CSV as the reference's CPU rows:

    python -m paper_2103_01216_b200.cli gen  --kind perm --n 1000000 --out h.u64
    python -m paper_2103_01216_b200.cli run  --algo rp --variant final --input h.u64 --verify
    python -m paper_2103_01216_b200.cli sweep --algo scan --n 1048576 4194304 --csv r.csv

Exit codes: 0 ok, 1 usage, 2 I/O, 3 verification failure.

Differences from the reference, all on purpose:
* inputs go ``.u64`` file -> pinned host memory -> device once; every rep
  runs on a fresh device copy of them and the timed region covers only the
  algorithm (device-synchronised on both sides), as the reference times only
  its body;
* the ``threads`` column is 0 for GPU rows (``--threads`` is accepted and
  ignored: the device decides its own parallelism);
* ``--verify`` checks with numpy on the host (cumsum, sort, mask, roll, the
  sequential swap order) — the reference's oracles in ``baselines.py`` —
  never with the library under test.
Registered: scan, scan-blocked, reduce, rotate, filter(-relaxed),
partition(-relaxed), quicksort(-relaxed), merge(-relaxed) and rp (all four
variants).  Algorithms outside this path (mergesort, sets, contraction,
graphs) are not registered here; asking for them is a usage error (exit 1).
"""
from __future__ import annotations

import argparse
import sys
import time
from dataclasses import dataclass

import numpy as np

from . import formats, pred, relaxed, strong
from .runtime import EpsilonConfig, Rng, SpaceMeter, meter_scope

M64 = (1 << 64) - 1
EVEN = pred.even()

ALGO_KIND = {
    "scan": "ints", "scan-blocked": "ints", "reduce": "ints", "rotate": "ints",
    "filter": "ints", "filter-relaxed": "ints",
    "partition": "ints", "partition-relaxed": "ints",
    "quicksort": "ints", "quicksort-relaxed": "ints",
    "merge": "ints", "merge-relaxed": "ints",
    "rp": "perm",
}
ALGORITHMS = sorted(ALGO_KIND)
GEN_KINDS = ("ints", "perm")


@dataclass
class BenchConfig:
    algo: str
    n: int
    epsilon: float = 0.5
    prefix_fraction: float = 0.02
    threads: int = 0
    seed: int = 1
    reps: int = 1
    verify: bool = False
    variant: str = "final"

    def budget(self) -> EpsilonConfig:
        return EpsilonConfig(self.epsilon, self.prefix_fraction)


def generate_input(kind: str, n: int, seed: int) -> np.ndarray:
    """Deterministic inputs, the reference's generators (cli.py:63-68)."""
    rng = Rng(seed)
    if kind == "ints":
        return rng.words(0, n)
    if kind == "perm":
        return relaxed.make_swap_sequence(n, rng)
    raise ValueError(f"unknown or off-path input kind {kind!r} (this path takes {GEN_KINDS})")


# ---------------------------------------------------------------------------
# host-side checks (numpy; the reference's sequential oracles)

def _ref_exclusive_scan(x: np.ndarray) -> tuple[np.ndarray, int]:
    if len(x) == 0:
        return x.copy(), 0
    inc = np.cumsum(x, dtype=np.uint64)
    exc = np.empty_like(inc)
    exc[0] = 0
    exc[1:] = inc[:-1]
    return exc, int(inc[-1])


def _ref_knuth(h: np.ndarray) -> np.ndarray:
    """The sequential swap order the rounds must reproduce: ids descending,
    swap A[i] with A[H[i]] (relaxed.py:64-70)."""
    a = np.arange(len(h), dtype=np.uint64)
    hh = h.astype(np.int64)
    for i in range(len(h) - 1, -1, -1):
        j = hh[i]
        if j != i:
            a[i], a[j] = a[j], a[i]
    return a


class _Run:
    def __init__(self, body, verify, rounds=None):
        self.body = body
        self.verify = verify
        self.rounds = rounds if rounds is not None else (lambda: 0)


def _sort_unsigned(t) -> None:
    """Sort a device int64 tensor as unsigned words (flip the sign bit around
    a signed sort)."""
    import torch

    sign = torch.tensor(-(1 << 63), dtype=torch.int64, device=t.device)
    t.bitwise_xor_(sign)
    t.copy_(torch.sort(t).values)
    t.bitwise_xor_(sign)


def _make_run(cfg: BenchConfig, dev_in, host_in: np.ndarray) -> _Run:
    import torch

    algo = cfg.algo
    budget = cfg.budget()
    a = dev_in.clone()
    state: dict = {}

    def host(t) -> np.ndarray:
        return t.cpu().numpy().view(np.uint64)

    if algo in ("scan", "scan-blocked"):
        fn = strong.scan if algo == "scan" else strong.scan_blocked

        def body():
            state["res"] = fn(a)

        def verify():
            ref, tot = _ref_exclusive_scan(host_in)
            return np.array_equal(host(a), ref) and state["res"].total == tot

        return _Run(body, verify)

    if algo == "reduce":
        return _Run(lambda: state.__setitem__("t", strong.reduce(a)),
                    lambda: state["t"] == int(np.sum(host_in, dtype=np.uint64)))

    if algo == "rotate":
        o = len(host_in) // 3
        return _Run(lambda: strong.rotate(a, o),
                    lambda: np.array_equal(host(a), np.roll(host_in, -o)))

    if algo in ("filter", "filter-relaxed"):
        def body():
            if algo == "filter":
                state["m"] = strong.filter_kway(a, EVEN)
            else:
                state["m"] = relaxed.filter_relaxed(a, EVEN, budget,
                                                    stats_sink=state.setdefault("s", []))

        def verify():
            ref = host_in[(host_in & np.uint64(1)) == 0]
            m = state["m"]
            return m == len(ref) and np.array_equal(host(a)[:m], ref)

        return _Run(body, verify,
                    lambda: state["s"][0].rounds if state.get("s") else 0)

    if algo in ("partition", "partition-relaxed"):  # cli.py:226-247
        def body():
            if algo == "partition":
                state["m"] = strong.partition_unstable(a, EVEN)
            else:
                state["m"] = relaxed.partition_relaxed(a, EVEN, budget,
                                                       stats_sink=state.setdefault("s", []))

        def verify():
            m, out = state["m"], host(a)
            ev = (out & np.uint64(1)) == 0
            return (m == int(np.count_nonzero((host_in & np.uint64(1)) == 0))
                    and bool(np.all(ev[:m])) and not bool(np.any(ev[m:]))
                    and np.array_equal(np.sort(out), np.sort(host_in)))

        return _Run(body, verify, lambda: state["s"][0].rounds if state.get("s") else 0)

    if algo in ("quicksort", "quicksort-relaxed"):  # cli.py:249-257
        rng = Rng(cfg.seed)
        fn = (lambda: strong.quicksort_strong(a, rng)) if algo == "quicksort" else \
             (lambda: relaxed.quicksort_relaxed(a, rng, budget))
        return _Run(fn, lambda: np.array_equal(host(a), np.sort(host_in)))

    if algo in ("merge", "merge-relaxed"):
        split = len(host_in) // 2
        if split:
            _sort_unsigned(a[:split])
        if len(host_in) - split:
            _sort_unsigned(a[split:])
        torch.cuda.synchronize()
        fn = (lambda: strong.merge_strong(a, split)) if algo == "merge" else \
             (lambda: relaxed.merge_relaxed(a, split, budget))
        return _Run(fn, lambda: np.array_equal(host(a), np.sort(host_in)))

    if algo == "rp":
        a = torch.arange(len(host_in), dtype=torch.int64, device=dev_in.device)

        def body():
            state["stats"] = relaxed.random_permutation(a, dev_in, cfg.variant, budget)

        return _Run(body, lambda: np.array_equal(host(a), _ref_knuth(host_in)),
                    lambda: state["stats"].rounds)

    raise ValueError(f"unknown algorithm {algo!r}")


def run_bench(cfg: BenchConfig, dev_in, host_in: np.ndarray) -> list[dict]:
    """Reps of one algorithm; timing covers only the algorithm body."""
    import torch

    rows = []
    for rep in range(cfg.reps):
        run = _make_run(cfg, dev_in, host_in)
        meter = SpaceMeter()
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        report = meter_scope(meter, 1 << 62, run.body)
        torch.cuda.synchronize()
        elapsed_ms = (time.perf_counter() - t0) * 1000.0
        verified = "skipped"
        if cfg.verify:
            verified = "true" if run.verify() else "false"
        rows.append({
            "algo": cfg.algo if cfg.algo != "rp" else f"rp-{cfg.variant}",
            "n": cfg.n, "epsilon": cfg.epsilon, "threads": 0, "seed": cfg.seed, "rep": rep,
            "time_ms": round(elapsed_ms, 3), "peak_heap_words": report.peak_words,
            "rounds": run.rounds(), "verified": verified,
        })
    return rows


# ---------------------------------------------------------------------------
# command line

class _Parser(argparse.ArgumentParser):
    def error(self, message):
        self.print_usage(sys.stderr)
        print(f"{self.prog}: error: {message}", file=sys.stderr)
        sys.exit(1)


def _normalize_algo(algo: str, variant: str | None) -> tuple[str, str]:
    if algo.startswith("rp-"):
        return "rp", algo[3:]
    return algo, variant or "final"


def build_parser() -> _Parser:
    p = _Parser(prog="pipal-gpu", description=__doc__.split("\n\n")[0])
    sub = p.add_subparsers(dest="command", required=True)
    g = sub.add_parser("gen", help="generate a deterministic input file")
    g.add_argument("--kind", required=True, choices=GEN_KINDS)
    g.add_argument("--n", required=True, type=int)
    g.add_argument("--seed", type=int, default=1)
    g.add_argument("--out", required=True)
    r = sub.add_parser("run", help="run one algorithm on the GPU")
    r.add_argument("--algo", required=True)
    r.add_argument("--input", required=True)
    r.add_argument("--epsilon", type=float, default=0.5)
    r.add_argument("--prefix-frac", type=float, default=0.02)
    r.add_argument("--threads", type=int, default=0)
    r.add_argument("--seed", type=int, default=1)
    r.add_argument("--reps", type=int, default=1)
    r.add_argument("--verify", action="store_true")
    r.add_argument("--csv")
    r.add_argument("--variant", choices=relaxed.RP_VARIANTS)
    s = sub.add_parser("sweep", help="cross parameter lists through run")
    s.add_argument("--algo", required=True)
    s.add_argument("--n", required=True, type=int, nargs="+")
    s.add_argument("--epsilon", type=float, nargs="+", default=[0.5])
    s.add_argument("--threads", type=int, nargs="+", default=[0])
    s.add_argument("--prefix-frac", type=float, default=0.02)
    s.add_argument("--seed", type=int, default=1)
    s.add_argument("--reps", type=int, default=1)
    s.add_argument("--verify", action="store_true")
    s.add_argument("--csv", required=True)
    s.add_argument("--variant", choices=relaxed.RP_VARIANTS)
    return p


def _cmd_gen(args) -> int:
    try:
        data = generate_input(args.kind, args.n, args.seed)
    except ValueError as exc:
        print(f"pipal-gpu gen: {exc}", file=sys.stderr)
        return 1
    try:
        formats.write_ints(args.out, data)
    except OSError as exc:
        print(f"pipal-gpu gen: cannot write {args.out}: {exc}", file=sys.stderr)
        return 2
    return 0


def _load_input(algo: str, path):
    """-> (device words, host numpy words); perm inputs are validated."""
    import torch

    kind = formats.kind_of_path(path)
    if kind != "ints":
        raise ValueError(f"{path}: holds a {kind!r} input but {algo} expects 'ints'")
    pinned = formats.read_ints_pinned(path)
    host = pinned.numpy().view(np.uint64)
    dev = pinned.to(torch.device("cuda", torch.cuda.current_device()), non_blocking=True)
    torch.cuda.synchronize()
    if ALGO_KIND[algo] == "perm":
        relaxed.validate_swap_sequence(dev)  # on the device (relaxed.py:55-58 semantics)
    return dev, host


def _cmd_run(args) -> int:
    algo, variant = _normalize_algo(args.algo, args.variant)
    if algo not in ALGO_KIND:
        print(f"pipal-gpu run: unknown or off-path algorithm {args.algo!r}", file=sys.stderr)
        return 1
    try:
        dev, host = _load_input(algo, args.input)
    except OSError as exc:
        print(f"pipal-gpu run: cannot read {args.input}: {exc}", file=sys.stderr)
        return 2
    except ValueError as exc:
        print(f"pipal-gpu run: {exc}", file=sys.stderr)
        return 1
    cfg = BenchConfig(algo=algo, n=len(host), epsilon=args.epsilon,
                      prefix_fraction=args.prefix_frac, seed=args.seed, reps=args.reps,
                      verify=args.verify, variant=variant)
    rows = run_bench(cfg, dev, host)
    for row in rows:
        print(",".join(str(row[c]) for c in formats.CSV_COLUMNS))
    if args.csv:
        try:
            formats.append_report_rows(args.csv, rows)
        except OSError as exc:
            print(f"pipal-gpu run: cannot write {args.csv}: {exc}", file=sys.stderr)
            return 2
    if args.verify and any(r["verified"] == "false" for r in rows):
        print("pipal-gpu run: verification FAILED", file=sys.stderr)
        return 3
    return 0


def _cmd_sweep(args) -> int:
    import torch

    algo, variant = _normalize_algo(args.algo, args.variant)
    if algo not in ALGO_KIND:
        print(f"pipal-gpu sweep: unknown or off-path algorithm {args.algo!r}", file=sys.stderr)
        return 1
    failed = False
    for n in args.n:
        try:
            host = generate_input(ALGO_KIND[algo], n, args.seed)
        except ValueError as exc:
            print(f"pipal-gpu sweep: {exc}", file=sys.stderr)
            return 1
        dev = torch.from_numpy(host.view(np.int64)).cuda()
        for eps in args.epsilon:
            for _threads in args.threads:
                cfg = BenchConfig(algo=algo, n=n, epsilon=eps, prefix_fraction=args.prefix_frac,
                                  seed=args.seed, reps=args.reps, verify=args.verify,
                                  variant=variant)
                rows = run_bench(cfg, dev, host)
                try:
                    formats.append_report_rows(args.csv, rows)
                except OSError as exc:
                    print(f"pipal-gpu sweep: cannot write {args.csv}: {exc}", file=sys.stderr)
                    return 2
                failed |= any(r["verified"] == "false" for r in rows)
    return 3 if failed else 0


def main(argv=None) -> int:
    args = build_parser().parse_args(argv)
    if args.command == "gen":
        return _cmd_gen(args)
    if args.command == "run":
        return _cmd_run(args)
    return _cmd_sweep(args)


if __name__ == "__main__":
    sys.exit(main())
