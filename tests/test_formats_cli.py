"""The .u64 container, the report CSV and the GPU command line
(reference formats.py and cli.py)."""
from __future__ import annotations

import struct

import numpy as np
import pytest

from paper_2103_01216_b200 import cli, formats
from paper_2103_01216_b200.runtime import Rng


def test_u64_roundtrip_and_layout(tmp_path):
    x = np.array([0, 1, (1 << 64) - 1, 12345678901234567], dtype=np.uint64)
    p = tmp_path / "x.u64"
    formats.write_ints(p, x)
    raw = p.read_bytes()
    # formats.py:25-30: magic, LE count, LE words
    assert raw[:8] == b"PIPU64\x00\x01"
    assert struct.unpack("<Q", raw[8:16])[0] == 4
    assert struct.unpack("<4Q", raw[16:]) == tuple(int(v) for v in x)
    assert np.array_equal(formats.read_ints(p), x)
    assert formats.kind_of_path(p) == "ints"


def test_u64_empty(tmp_path):
    p = tmp_path / "e.u64"
    formats.write_ints(p, np.empty(0, dtype=np.uint64))
    assert len(formats.read_ints(p)) == 0


@pytest.mark.parametrize("blob,msg", [(b"NOTMAGIC" + b"\0" * 8, "unrecognized file magic"),
                                      (b"PIPLST\x00\x01" + struct.pack("<Q", 0), "not an integer file"),
                                      (b"PIPU64\x00\x01" + struct.pack("<Q", 3) + b"\0" * 16, "truncated"),
                                      (b"PIPU64\x00\x01", "truncated")])
def test_u64_errors(tmp_path, blob, msg):
    p = tmp_path / "bad.u64"
    p.write_bytes(blob)
    with pytest.raises(ValueError, match=msg):
        formats.read_ints(p)


def test_report_csv_schema(tmp_path):
    p = tmp_path / "r.csv"
    row = {"algo": "scan", "n": 8, "epsilon": 0.5, "threads": 0, "seed": 1, "rep": 0,
           "time_ms": 1.5, "peak_heap_words": 0, "rounds": 0, "verified": "true"}
    formats.append_report_rows(p, [row])
    formats.append_report_rows(p, [dict(row, rep=1, verified="skipped")])
    rows = formats.check_report_csv(p)
    assert [r["rep"] for r in rows] == [0, 1]
    assert p.read_text().splitlines()[0] == ",".join(formats.CSV_COLUMNS)
    bad = tmp_path / "bad.csv"
    bad.write_text(p.read_text().replace("skipped", "maybe"))
    with pytest.raises(ValueError, match="bad verified flag"):
        formats.check_report_csv(bad)


def test_report_csv_matches_reference(ref):
    # same column list as the reference's formats.py:33-34
    import pipal.formats as rf

    assert rf.CSV_COLUMNS == formats.CSV_COLUMNS
    assert rf.MAGIC == formats.MAGIC


def test_reference_reads_our_file(ref, tmp_path):
    import pipal.formats as rf

    x = Rng(3).words(0, 1000)
    p = tmp_path / "x.u64"
    formats.write_ints(p, x)
    assert np.array_equal(rf.read_ints(p), x)
    q = tmp_path / "y.u64"
    rf.write_ints(q, x)
    assert np.array_equal(formats.read_ints(q), x)


@pytest.mark.parametrize("kind", ["ints", "perm"])
def test_cli_gen(tmp_path, kind):
    p = tmp_path / f"{kind}.u64"
    assert cli.main(["gen", "--kind", kind, "--n", "1000", "--seed", "7", "--out", str(p)]) == 0
    assert np.array_equal(formats.read_ints(p), cli.generate_input(kind, 1000, 7))


def test_cli_gen_matches_reference_generators(ref):
    from pipal import cli as rcli
    from pipal.runtime import Rng as RRng

    assert np.array_equal(cli.generate_input("ints", 5000, 4), rcli.gen_ints(5000, RRng(4)))
    assert np.array_equal(cli.generate_input("perm", 5000, 4), rcli.gen_perm(5000, RRng(4)))


def test_cli_usage_errors(tmp_path, capsys):
    p = tmp_path / "x.u64"
    formats.write_ints(p, np.arange(10, dtype=np.uint64))
    assert cli.main(["run", "--algo", "mergesort", "--input", str(p)]) == 1
    assert cli.main(["run", "--algo", "scan", "--input", str(tmp_path / "missing.u64")]) == 2
    lst = tmp_path / "l.u64"
    lst.write_bytes(b"PIPLST\x00\x01" + struct.pack("<Q", 0))
    assert cli.main(["run", "--algo", "scan", "--input", str(lst)]) == 1
    assert cli.main(["gen", "--kind", "ints", "--n", "4", "--out", str(tmp_path / "no" / "x.u64")]) == 2
    with pytest.raises(SystemExit) as e:
        cli.main(["gen", "--kind", "tree", "--n", "5", "--out", str(p)])
    assert e.value.code == 1


def test_cli_reference_swap_order(orc):
    # the CLI's numpy check applies swaps in the order the oracle does
    h = cli.generate_input("perm", 3000, 11)
    want = np.arange(3000, dtype=np.uint64)
    orc.seq_knuth_shuffle(want, h)
    assert np.array_equal(cli._ref_knuth(h), want)


ALGOS = ["scan", "scan-blocked", "reduce", "rotate", "filter", "filter-relaxed", "partition",
         "partition-relaxed", "quicksort", "quicksort-relaxed", "merge", "merge-relaxed",
         "rp-naive", "rp-flat", "rp-oneres", "rp-final"]


@pytest.mark.gpu
@pytest.mark.parametrize("algo", ALGOS)
def test_cli_run_verify(tmp_path, algo):
    kind = "perm" if algo.startswith("rp") else "ints"
    p = tmp_path / "in.u64"
    assert cli.main(["gen", "--kind", kind, "--n", "100003", "--seed", "5", "--out", str(p)]) == 0
    csvp = tmp_path / "r.csv"
    assert cli.main(["run", "--algo", algo, "--input", str(p), "--verify", "--reps", "2",
                     "--csv", str(csvp)]) == 0
    rows = formats.check_report_csv(csvp)
    assert len(rows) == 2 and all(r["verified"] == "true" for r in rows)
    assert rows[0]["algo"] == algo and rows[0]["n"] == 100003 and rows[0]["threads"] == 0
    if algo.startswith("rp"):
        assert rows[0]["rounds"] > 0 and rows[0]["peak_heap_words"] > 0


@pytest.mark.gpu
def test_cli_sweep_and_pinned_read(tmp_path):
    csvp = tmp_path / "s.csv"
    assert cli.main(["sweep", "--algo", "filter-relaxed", "--n", "1000", "70000",
                     "--epsilon", "0.5", "0.7", "--verify", "--csv", str(csvp)]) == 0
    rows = formats.check_report_csv(csvp)
    assert len(rows) == 4 and all(r["verified"] == "true" for r in rows)
    assert all(r["rounds"] >= 1 for r in rows)
    x = Rng(9).words(0, 12345)
    p = tmp_path / "x.u64"
    formats.write_ints(p, x)
    t = formats.read_ints_pinned(p)
    assert t.is_pinned() and np.array_equal(t.numpy().view(np.uint64), x)
    d = formats.read_ints_device(p)
    assert d.is_cuda and np.array_equal(d.cpu().numpy().view(np.uint64), x)
