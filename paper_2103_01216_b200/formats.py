"""The ``.u64`` input container and the benchmark report CSV.

Mirrors the reference's ``formats.py`` for the integer kind it uses on this
path (``formats.py:25-30`` magic table, ``:67-76`` read/write, ``:33-34`` CSV
columns, ``:124-158`` report writer/checker): a file is the 8-byte magic
``PIPU64\\0\\x01``, a little-endian u64 count, then that many little-endian u64
words.  The other kinds (list/tree/graph) are recognised by their magic but
belong to subsystems outside this path and are rejected with ``ValueError``.

``read_ints_pinned`` reads the words straight into page-locked host memory
(one ``readinto`` — no intermediate copy), ready for an asynchronous
host-to-device copy; ``read_ints_device`` goes on to the GPU.
"""
from __future__ import annotations

import csv
import struct
from pathlib import Path

import numpy as np

__all__ = ["MAGIC", "CSV_COLUMNS", "write_ints", "read_ints", "read_ints_pinned",
           "read_ints_device", "kind_of_path", "append_report_rows", "check_report_csv"]

MAGIC = {
    "ints": b"PIPU64\x00\x01",
    "list": b"PIPLST\x00\x01",
    "tree": b"PIPTRE\x00\x01",
    "graph": b"PIPGRP\x00\x01",
}
_KIND = {v: k for k, v in MAGIC.items()}
_HEADER = 16  # magic + count

CSV_COLUMNS = ["algo", "n", "epsilon", "threads", "seed", "rep",
               "time_ms", "peak_heap_words", "rounds", "verified"]


def _kind(f, path) -> str:
    kind = _KIND.get(f.read(8))
    if kind is None:
        raise ValueError(f"{path}: unrecognized file magic")
    return kind


def kind_of_path(path) -> str:
    with open(path, "rb") as f:
        return _kind(f, path)


def _open_ints(f, path) -> int:
    if _kind(f, path) != "ints":
        raise ValueError(f"{path}: not an integer file")
    raw = f.read(8)
    if len(raw) != 8:
        raise ValueError(f"{path}: truncated file")
    (n,) = struct.unpack("<Q", raw)
    return n


def write_ints(path, words) -> None:
    words = np.ascontiguousarray(words)
    with open(path, "wb") as f:
        f.write(MAGIC["ints"])
        f.write(struct.pack("<Q", len(words)))
        f.write(words.astype("<u8", copy=False).tobytes())


def read_ints(path) -> np.ndarray:
    with open(path, "rb") as f:
        n = _open_ints(f, path)
        out = np.empty(n, dtype=np.uint64)
        got = f.readinto(memoryview(out.view(np.uint8)))
        if got != 8 * n:
            raise ValueError(f"{path}: truncated file")
    if np.little_endian:
        return out
    return out.byteswap()


def read_ints_pinned(path):
    """Read a ``.u64`` file into a page-locked int64 torch tensor (u64 bits)."""
    import torch

    with open(path, "rb") as f:
        n = _open_ints(f, path)
        host = torch.empty(n, dtype=torch.int64, pin_memory=True)
        if n:
            got = f.readinto(memoryview(host.numpy().view(np.uint8)))
            if got != 8 * n:
                raise ValueError(f"{path}: truncated file")
    return host


def read_ints_device(path, device=None):
    """``.u64`` file -> pinned host -> device words (int64 tensor, u64 bits)."""
    import torch

    host = read_ints_pinned(path)
    dev = torch.device("cuda", torch.cuda.current_device() if device is None else device)
    out = torch.empty_like(host, device=dev)
    out.copy_(host, non_blocking=True)
    torch.cuda.current_stream(dev).synchronize()
    return out


def append_report_rows(path, rows: list[dict]) -> None:
    """Append rows to the report CSV, writing the header on first use."""
    path = Path(path)
    fresh = not path.exists() or path.stat().st_size == 0
    with open(path, "a", newline="") as f:
        w = csv.DictWriter(f, fieldnames=CSV_COLUMNS)
        if fresh:
            w.writeheader()
        for row in rows:
            w.writerow({k: row[k] for k in CSV_COLUMNS})


def check_report_csv(path) -> list[dict]:
    """Parse and validate a report: the reference's fixed, fully typed schema."""
    with open(path, newline="") as f:
        reader = csv.DictReader(f)
        if reader.fieldnames != CSV_COLUMNS:
            raise ValueError(f"{path}: unexpected CSV columns {reader.fieldnames}")
        rows = []
        for row in reader:
            parsed = {"algo": row["algo"], "n": int(row["n"]), "epsilon": float(row["epsilon"]),
                      "threads": int(row["threads"]), "seed": int(row["seed"]),
                      "rep": int(row["rep"]), "time_ms": float(row["time_ms"]),
                      "peak_heap_words": int(row["peak_heap_words"]),
                      "rounds": int(row["rounds"]), "verified": row["verified"]}
            if parsed["verified"] not in ("true", "false", "skipped"):
                raise ValueError(f"{path}: bad verified flag {row['verified']!r}")
            rows.append(parsed)
        return rows
