"""The device deterministic-reservations engine: ReservationTable,
run_rounds / RoundView and runtime.compact_by_mask.

* the reference's own scenarios (tests/test_detres.py of the reference:
  put/get, batched duplicates, sequential max-map equality, the load cap,
  delete, clear, metering, and the run_rounds client mocks of :115-194),
  restated with the client callbacks working on CUDA tensors;
* golden fixtures made by the reference itself (tests/golden/detres.npz):
  the table's SLOT LAYOUT (which key sits in which slot, with which value)
  after seeded batches and after a delete, and compact_by_mask outputs.

Reference: detres.py:40-307, runtime.py:335-355.
"""
from __future__ import annotations

import numpy as np
import pytest

from conftest import golden

pytestmark = pytest.mark.gpu
NIL = (1 << 64) - 1


@pytest.fixture(scope="module")
def dr():
    from paper_2103_01216_b200 import detres

    return detres


def words(vals):
    return np.array(vals, dtype=np.uint64)


# ---------------------------------------------------------------- table

def test_put_then_get(dr):
    t = dr.ReservationTable(16)
    dr.reserve_max(t, 3, 7)
    assert t.get(3) == 7
    assert t.get(4) is None


def test_max_semantics_batched_duplicates(dr):
    t = dr.ReservationTable(16)
    t.reserve_max(words([5, 5, 5]), words([3, 9, 5]))
    assert t.get(5) == 9
    t.put_max(5, 4)
    assert t.get(5) == 9
    t.put_max(5, 11)
    assert t.get(5) == 11


def test_table_matches_sequential_max_map(dr):
    rng = np.random.default_rng(42)
    keys = rng.integers(0, 500, size=10_000, dtype=np.uint64)
    vals = rng.integers(0, 1 << 63, size=10_000, dtype=np.uint64)
    ref: dict[int, int] = {}
    for k, v in zip(keys.tolist(), vals.tolist()):
        ref[k] = max(ref.get(k, 0), v)
    t = dr.ReservationTable(2048)
    for s in range(0, 10_000, 700):
        t.reserve_max(keys[s:s + 700], vals[s:s + 700])
    got, found = t.lookup(np.arange(500, dtype=np.uint64))
    for k in range(500):
        if k in ref:
            assert found[k] and int(got[k]) == ref[k]
        else:
            assert not found[k]


def test_load_factor_capped_at_half(dr):
    t = dr.ReservationTable(64)
    t.reserve_max(np.arange(32, dtype=np.uint64), np.arange(32, dtype=np.uint64))
    assert t.peak_load <= 0.5
    with pytest.raises(RuntimeError, match="overfull"):
        t.reserve_max(np.arange(32, 64, dtype=np.uint64), np.arange(32, dtype=np.uint64))


def test_delete_then_empty(dr):
    t = dr.ReservationTable(32)
    keys = words([1, 9, 17, 25, 33])
    t.reserve_max(keys, keys)
    t.delete(keys)
    assert t.count == 0
    _, found = t.lookup(keys)
    assert not found.any()


def test_clear_resets_all_slots(dr):
    t = dr.ReservationTable(32)
    t.reserve_max(words([2, 4, 6]), words([1, 1, 1]))
    t.clear()
    assert t.count == 0
    _, found = t.lookup(words([2, 4, 6]))
    assert not found.any()


def test_table_property_vs_dict(dr):
    rng = np.random.default_rng(5)
    for trial in range(40):
        m = int(rng.integers(0, 200))
        pairs = [(int(rng.integers(0, 41)), int(rng.integers(0, 1001))) for _ in range(m)]
        t = dr.ReservationTable(256)
        ref: dict[int, int] = {}
        if pairs:
            t.reserve_max(words([k for k, _ in pairs]), words([v for _, v in pairs]))
            for k, v in pairs:
                ref[k] = max(ref.get(k, 0), v)
        got, found = t.lookup(np.arange(41, dtype=np.uint64))
        for k in range(41):
            assert (int(got[k]) if found[k] else None) == ref.get(k), (trial, k)


def test_table_charges_meter(dr):
    from paper_2103_01216_b200.runtime import SpaceMeter, metered

    meter = SpaceMeter()
    with metered(meter):
        t = dr.ReservationTable(512)
        assert meter.current_words == 2 * 512
        t.release()
    assert meter.current_words == 0


def test_table_device_tensors_in_and_out(dr):
    import torch

    t = dr.ReservationTable(1 << 12)
    k = torch.arange(0, 3000, 3, dtype=torch.int64, device="cuda")
    t.reserve_max(k, k * 2)
    v, f = t.lookup(torch.arange(0, 3000, dtype=torch.int64, device="cuda"))
    assert v.is_cuda and f.is_cuda
    assert bool(f[::3].all()) and not bool(f[1::3].any())
    assert torch.equal(v[::3], k * 2)


@pytest.mark.parametrize("case", ["small", "collide", "batches", "dense"])
def test_table_slot_layout_equals_reference(dr, case):
    g = golden("detres")
    cap, nb, count = (int(x) for x in g[f"{case}_cap"])
    t = dr.ReservationTable(cap)
    for i in range(nb):
        t.reserve_max(g[f"{case}_k{i}"], g[f"{case}_v{i}"])
    assert t.count == count
    assert t.peak_load == pytest.approx(float(g[f"{case}_peak"][0]))
    keys = t.slot_keys()
    assert np.array_equal(keys, g[f"{case}_keys"])
    vals = t.vals.cpu().numpy().view(np.uint64)
    occ = keys != np.uint64(NIL)
    assert np.array_equal(np.where(occ, vals, 0).astype(np.uint64), g[f"{case}_vals"])
    t.delete(g[f"{case}_delk"])
    assert np.array_equal(t.slot_keys(), g[f"{case}_keys_after_delete"])
    assert t.count == int(g[f"{case}_count_after_delete"][0])


# ---------------------------------------------------------------- compact_by_mask

@pytest.mark.parametrize("n", [1, 255, 256, 257, 10_000, 20_011])
def test_compact_by_mask_golden(n):
    import torch

    from paper_2103_01216_b200.runtime import compact_by_mask

    g = golden("detres")
    a, keep, want = g[f"compact_in_{n}"], g[f"compact_keep_{n}"], g[f"compact_out_{n}"]
    b = a.copy()
    assert compact_by_mask(b, keep, n) == len(want)
    assert np.array_equal(b[: len(want)], want)
    t = torch.from_numpy(a.view(np.int64).copy()).cuda()
    m = compact_by_mask(t, torch.from_numpy(keep).cuda(), n)
    assert m == len(want) and np.array_equal(t[:m].cpu().numpy().view(np.uint64), want)


def test_compact_by_mask_large_and_partial(orc):
    import torch

    from paper_2103_01216_b200.runtime import compact_by_mask

    rng = np.random.default_rng(3)
    for n in (3_000_017, 1 << 22):
        a = rng.integers(0, 1 << 64, size=n, dtype=np.uint64)
        keep = rng.random(n) < 0.5
        t = torch.from_numpy(a.view(np.int64).copy()).cuda()
        k = torch.from_numpy(keep).cuda()
        m = compact_by_mask(t, k, n - 5)  # only a[0:n-5)
        want = a[: n - 5][keep[: n - 5]]
        assert m == len(want) and np.array_equal(t[:m].cpu().numpy().view(np.uint64), want)
        # odd offsets: unaligned words and flags take the scalar path
        t = torch.from_numpy(a.view(np.int64).copy()).cuda()
        m = compact_by_mask(t[1:], k[1:], n - 1)
        want = a[1:][keep[1:]]
        assert m == len(want) and np.array_equal(t[1:1 + m].cpu().numpy().view(np.uint64), want)


# ---------------------------------------------------------------- run_rounds

def _client_all_succeed():
    def reserve(view):
        pass

    def commit(view):
        view.committed[:] = True

    def clean(view):
        pass

    return reserve, commit, clean


def test_all_commits_two_rounds(dr):
    r, c, cl = _client_all_succeed()
    stats = dr.run_rounds(8, 4, r, c, cl)
    assert stats.rounds == 2
    assert stats.committed_per_round == [4, 4]


def test_single_iterate_single_round(dr):
    r, c, cl = _client_all_succeed()
    stats = dr.run_rounds(1, 4, r, c, cl)
    assert stats.rounds == 1 and stats.committed_per_round == [1]


def test_conservation_and_packing_order(dr):
    import torch

    n = 1000
    seen: list[torch.Tensor] = []
    retried = torch.zeros(n, dtype=torch.bool, device="cuda")

    def reserve(view):
        pass

    def commit(view):
        ids = view.ids
        ok = (ids % 2 == 0) | retried[ids]
        view.committed[:] = ok
        seen.append(ids[ok].clone())
        retried[ids] = True

    def clean(view):
        assert bool((view.ids[1:] > view.ids[:-1]).all())  # packed order: ascending

    stats = dr.run_rounds(n, 128, reserve, commit, clean)
    assert sorted(torch.cat(seen).tolist()) == list(range(n))
    assert stats.total_committed == n


def test_livelock_guard_aborts(dr):
    def nothing(view):
        pass

    def commit(view):
        view.committed[:] = False

    with pytest.raises(dr.LivelockError):
        dr.run_rounds(10, 4, nothing, commit, nothing)


def test_trace_collects_committed_ids(dr):
    trace: list = []

    def commit(view):
        view.committed[:] = (view.ids % 3 != 0) | (view.round_index > 0)

    def other(view):
        pass

    dr.run_rounds(9, 9, other, commit, other, trace=trace)
    assert sorted(trace[0].tolist()) == [1, 2, 4, 5, 7, 8]
    assert sorted(trace[1].tolist()) == [0, 3, 6]


def test_run_rounds_with_table_client_is_knuth_shuffle(dr, orc):
    """A full DR client on the generic engine: the reference's 'final'
    permutation rules (relaxed.py:130-197: reserve R[H[i]] = max i, commit
    iff i owns its own slot and its target) on a device ReservationTable,
    ids descending from n-1 (relaxed.py:107-120).  The result must equal the
    sequential Knuth shuffle and the rounds the oracle's port."""
    import torch

    from paper_2103_01216_b200.relaxed import make_swap_sequence
    from paper_2103_01216_b200.runtime import EpsilonConfig, Rng

    n = 20_000
    h_np = make_swap_sequence(n, Rng(9))
    a = torch.arange(n, dtype=torch.int64, device="cuda")
    h = torch.from_numpy(h_np.view(np.int64)).cuda()
    nonself = torch.nonzero(h != torch.arange(n, device="cuda")).flatten().flip(0)
    prefix = EpsilonConfig(0.5).prefix_words(n)
    table = dr.ReservationTable(4 * prefix)
    state = {"next": 0}

    def source(count):
        lo = state["next"]
        hi = min(lo + count, nonself.numel())
        state["next"] = hi
        return nonself[lo:hi]

    def reserve(view):
        ids = view.ids
        table.reserve_max(torch.cat([ids, h[ids]]), torch.cat([ids, ids]))

    def commit(view):
        ids = view.ids
        v_own, _ = table.lookup(ids)
        v_tgt, _ = table.lookup(h[ids])
        ok = (v_own == ids) & (v_tgt == ids)
        view.committed[:] = ok
        i, t = ids[ok], h[ids[ok]]
        ai, at = a[i].clone(), a[t].clone()
        a[i] = at
        a[t] = ai

    def clean(view):
        table.clear()

    st = dr.run_rounds(nonself.numel(), prefix, reserve, commit, clean, id_source=source)
    want = np.arange(n, dtype=np.uint64)
    orc.seq_knuth_shuffle(want, h_np)
    assert np.array_equal(a.cpu().numpy().view(np.uint64), want)
    info = orc.ref_random_permutation(np.arange(n, dtype=np.uint64), h_np, prefix, "naive")
    assert st.rounds == info["rounds"]
    assert st.committed_per_round == info["committed_per_round"]


def test_table_grow_and_numpy_source(dr):
    t = dr.ReservationTable(8)
    t.grow(100)
    assert t.capacity == 128
    t.put_max(7, 3)
    with pytest.raises(RuntimeError, match="only grow while empty"):
        t.grow(1000)

    # an id source that hands out numpy words (the reference's own clients do)
    state = {"next": 0}

    def source(count):
        lo = state["next"]
        hi = min(lo + count, 50)
        state["next"] = hi
        return np.arange(lo, hi, dtype=np.uint64)

    def nothing(view):
        pass

    def commit(view):
        view.committed[:] = (view.ids % 2 == 0) | (view.round_index > 0)

    trace: list = []
    st = dr.run_rounds(50, 16, nothing, commit, nothing, id_source=source, trace=trace)
    assert sorted(int(x) for tr in trace for x in tr.tolist()) == list(range(50))
    assert st.total_committed == 50


def test_compact_by_mask_uint8_flags_and_meter():
    import torch

    from paper_2103_01216_b200.runtime import SpaceMeter, compact_by_mask, metered

    x = np.arange(10_000, dtype=np.uint64)
    keep = (np.arange(10_000) % 7 == 3).astype(np.uint8) * 5  # any nonzero byte keeps
    t = torch.from_numpy(x.view(np.int64).copy()).cuda()
    meter = SpaceMeter()
    with metered(meter):
        m = compact_by_mask(t, torch.from_numpy(keep).cuda())
    assert meter.peak_words == 0  # zero heap, like the reference's (runtime.py:335-355)
    assert m == int((keep != 0).sum())
    assert np.array_equal(t[:m].cpu().numpy().view(np.uint64), x[keep != 0])
