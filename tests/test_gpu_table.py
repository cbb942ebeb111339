"""GPU parity of the HBM-resident table (C ABI, one rank) against the oracle.

Mirrors the reference's device-table / HbmTier unit tests
(proj/tests/test_device_table.cpp, test_hbm_ps.cpp) on the CUDA path:
bit-exact slot layout, pulled rows, additive push/drain, carry-over and the
error contract.
"""
import numpy as np
import pytest

from native import EMPTY

pytestmark = pytest.mark.gpu


def _tier(pkg, width=2, **kw):
    kw.setdefault("max_batch_keys", 1 << 18)
    kw.setdefault("max_working_set", 1 << 18)
    return pkg.Tier(width=width, **kw)


@pytest.mark.parametrize("n", [0, 1, 6, 7, 100, 5000, 150000])
def test_build_slot_layout_equals_ascending_insert(pkg, oracle, n):
    """device_table.hpp:51-73 inserted in ascending order (hbm_ps.hpp:89-98)."""
    rng = np.random.default_rng(n + 1)
    keys = rng.integers(0, 1 << 40, size=n, dtype=np.uint64)
    keys = np.concatenate([keys, keys[: n // 3]])  # duplicates are merged
    rng.shuffle(keys)
    t = _tier(pkg, width=4)
    rows = (keys.astype(np.float64)[:, None] * np.arange(1, 5)).astype(np.float32)
    t.build(keys, rows)
    uk = np.unique(keys)
    want = oracle.table_build(uk)
    slots, vals = t.table_slots(with_rows=True)
    assert slots.size == want.size == oracle.capacity(uk.size)
    assert np.array_equal(slots, want)
    live = slots != EMPTY
    exp = (slots[live].astype(np.float64)[:, None] * np.arange(1, 5)).astype(np.float32)
    assert np.array_equal(vals[live], exp)
    cap, occ, w = t.table_info()
    assert (cap, occ, w) == (want.size, uk.size, 4)
    t.close()


def test_capacity_rule_matches_reference(pkg):
    """test_device_table.cpp:33-47: 6 keys -> capacity 8."""
    t = _tier(pkg, width=1)
    t.build(np.arange(6, dtype=np.uint64), np.arange(6, dtype=np.float32))
    assert t.table_info()[:2] == (8, 6)
    t.build(np.empty(0, np.uint64))
    assert t.table_info()[:2] == (1, 0)  # empty table (test_device_table.cpp:49-54)
    t.close()


def test_pull_rows_bit_identical_any_order(pkg):
    rng = np.random.default_rng(7)
    keys = np.unique(rng.integers(0, 10**7, size=20000, dtype=np.uint64))
    rows = rng.standard_normal((keys.size, 8)).astype(np.float32)
    t = _tier(pkg, width=8)
    t.build(keys, rows)
    q = rng.choice(keys, size=30000)  # unsorted, with repeats
    got = t.pull(q)
    idx = np.searchsorted(keys, q)
    assert np.array_equal(got, rows[idx])
    again = t.pull(q)  # non-mutating (test_hbm_ps.cpp:131-133)
    assert np.array_equal(again, got)
    t.close()


def test_pull_missing_key_is_an_error(pkg):
    t = _tier(pkg, width=1)
    t.build(np.array([0, 1, 2, 3], np.uint64), np.arange(4, dtype=np.float32))
    with pytest.raises(pkg.Error) as e:
        t.pull(np.array([9], np.uint64))
    assert "missing key 9" in str(e.value)
    t.close()


def test_not_built_is_an_error(pkg):
    t = _tier(pkg, width=1)
    with pytest.raises(pkg.Error) as e:
        t.pull(np.array([1], np.uint64))
    assert "tables not built" in str(e.value)
    t.close()


def test_accumulate_is_elementwise_add(pkg):
    """test_device_table.cpp:64-74."""
    h = pkg.HbmTier(pkg.Topology(1, 1), 2)
    h.build_all([[11]], lambda k: [1.0, 1.0])
    h.accumulate({11: [0.5, -0.5]})
    assert h.get([11])[11] == [1.5, 0.5]
    h.accumulate({11: [0.0, 0.0]})
    assert h.table_at().get(11) == [1.5, 0.5]
    h.close()


def test_push_then_drain_is_exact_and_fifo(pkg):
    """test_hbm_ps.cpp:157-177 (one rank): 400 pushes of +1 per key."""
    h = pkg.HbmTier(pkg.Topology(1, 1), 1)
    h.build_all([[0, 1]], lambda k: [0.0])
    for n in range(800):
        h.push_deltas({n % 2: [1.0]})
    h.drain_accums()
    assert h.get([0, 1]) == {0: [400.0], 1: [400.0]}
    h.close()


def test_accumulate_missing_key_is_an_error(pkg):
    h = pkg.HbmTier(pkg.Topology(1, 1), 2)
    h.build_all([[0, 1]], lambda k: [0.0, 0.0])
    with pytest.raises(pkg.Error) as e:
        h.accumulate({7: [0.0, 0.0]})
    assert "accumulate to missing key 7" in str(e.value)
    h.close()


def test_carry_over_keeps_device_values(pkg):
    """test_hbm_ps.cpp:104-116 on one device."""
    h = pkg.HbmTier(pkg.Topology(1, 1), 1)
    h.build_all([[2, 3]], lambda k: [float(k)])
    h.accumulate({2: [10.0]})
    h.build_all([[2, 5]], lambda k: [float(k)])  # host would supply stale 2.0
    t = h.table_at()
    assert t.get(2) == [12.0]
    assert t.get(5) == [5.0]
    assert not t.contains(3)
    h.close()


def test_get_is_order_normalized(pkg):
    h = pkg.HbmTier(pkg.Topology(1, 1), 1)
    h.build_all([[0, 1, 2, 3]], lambda k: [float(k)])
    view = h.get([3, 0, 1])
    assert list(view.keys()) == [0, 1, 3]
    assert view[3] == [3.0]
    h.close()


def test_dump_is_sorted_and_complete(pkg):
    rng = np.random.default_rng(3)
    keys = rng.integers(0, 1 << 30, size=3000, dtype=np.uint64)
    t = _tier(pkg, width=4)
    rows = rng.standard_normal((keys.size, 4)).astype(np.float32)
    t.build(keys, rows)
    dk, dr = t.dump()
    uk, first = np.unique(keys, return_index=True)
    assert np.array_equal(dk, uk)
    # duplicates in the input: the staged row of the first occurrence wins
    assert np.array_equal(dr, rows[first])
    t.close()


def test_single_replica_sync_is_untouched(pkg):
    """test_hbm_ps.cpp:194-202."""
    t = _tier(pkg, width=1)
    out = t.dense_sync(np.array([3.25, -1.5], np.float32), deterministic=True)
    assert out.tolist() == [3.25, -1.5]
    t.close()
