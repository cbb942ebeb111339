"""CPU: parameter files in the reference's SSD-PS on-disk format (SURVEY §8(f)
row 3; ssd_ps.hpp:50-56). The writer must produce the reference SsdStore's
bytes exactly (SsdStore::dump, ssd_ps.hpp:229-243), the reader must apply
read_file_at's checks (ssd_ps.hpp:495-520), and the reference store must
recover, load and fsck our files (ssd_ps.hpp:294-340, 360-390).

Host-only entry points of libhps_gpu.so: no GPU needed. The GPU export of a
trained table is in test_gpu_train.py."""
import os
import zlib

import numpy as np
import pytest

from native import RefLib


@pytest.fixture(scope="module")
def ref():
    return RefLib()


def records(n, width, seed, opt=True):
    rng = np.random.default_rng(seed)
    keys = np.unique(rng.integers(0, 2**63, size=n, dtype=np.uint64))
    emb = rng.standard_normal((keys.size, width)).astype(np.float32)
    emb[::7] = -0.0  # signed zero must survive bit for bit
    o = rng.standard_normal((keys.size, width)).astype(np.float32) if opt else None
    return keys, emb, o


def files_of(d):
    return sorted(f for f in os.listdir(d) if f.startswith("pf_"))


def test_crc32_is_zlib(pkg):
    rng = np.random.default_rng(3)
    for n in (0, 1, 7, 8, 9, 1000, 65537):
        b = rng.integers(0, 256, n, dtype=np.uint8).tobytes()
        assert pkg.hps.crc32(b) == zlib.crc32(b)
        assert pkg.hps.crc32(b[n // 2:], pkg.hps.crc32(b[:n // 2])) == zlib.crc32(b)


@pytest.mark.parametrize("n,width,cap,opt", [
    (1, 1, 4096, False), (10000, 8, 4096, True), (4096, 16, 4096, False),
    (4097, 16, 4096, True), (3000, 64, 1000, True), (5, 3, 1, False),
])
def test_files_are_byte_identical_to_the_reference(pkg, ref, tmp_path, n, width, cap, opt):
    keys, emb, o = records(n, width, seed=n + width, opt=opt)
    ours, theirs = tmp_path / "ours", tmp_path / "ref"
    ours.mkdir()
    nf = pkg.hps.write_param_files(str(ours), keys, emb, o, file_capacity=cap)
    ref.store_dump(str(theirs), keys, emb, o, file_capacity=cap)
    assert nf == -(-keys.size // cap)
    assert files_of(ours) == files_of(theirs) == sorted(f"pf_{i}.bin" for i in range(nf))
    for f in files_of(ours):
        assert (ours / f).read_bytes() == (theirs / f).read_bytes(), f


def test_reference_store_recovers_loads_and_fscks_our_files(pkg, ref, tmp_path):
    keys, emb, o = records(20000, 16, seed=5)
    half = keys.size // 2
    # two exports with disjoint id ranges (two ranks) into one directory
    nf0 = pkg.hps.write_param_files(str(tmp_path), keys[:half], emb[:half], o[:half],
                                    file_capacity=2048, first_id=0)
    nf1 = pkg.hps.write_param_files(str(tmp_path), keys[half:], emb[half:], o[half:],
                                    file_capacity=2048, first_id=1000)
    assert not [f for f in os.listdir(tmp_path) if f.endswith(".tmp")]
    k, e, oo, info = ref.store_load_all(str(tmp_path), 16, keys.size, infer_width=True)
    assert np.array_equal(k, keys)
    assert e.tobytes() == emb.tobytes() and oo.tobytes() == o.tobytes()
    assert info == {"files": nf0 + nf1, "live_records": keys.size, "stale_records": 0,
                    "fsck_ok": 1, "fsck_files": nf0 + nf1, "recovered_invalid": 0}


def test_reader_round_trips_reference_files(pkg, ref, tmp_path):
    keys, emb, o = records(5000, 8, seed=9)
    ref.store_dump(str(tmp_path), keys, emb, o, file_capacity=4096)
    got = [pkg.hps.read_param_file(str(tmp_path / f)) for f in ("pf_0.bin", "pf_1.bin")]
    k = np.concatenate([g[0] for g in got])
    assert np.array_equal(k, keys)
    assert np.concatenate([g[1] for g in got]).tobytes() == emb.tobytes()
    assert np.concatenate([g[2] for g in got]).tobytes() == o.tobytes()


def test_zero_opt_state_when_absent(pkg, tmp_path):
    keys, emb, _ = records(100, 4, seed=1, opt=False)
    pkg.hps.write_param_files(str(tmp_path), keys, emb)
    k, e, o = pkg.hps.read_param_file(str(tmp_path / "pf_0.bin"))
    assert np.array_equal(k, keys) and e.tobytes() == emb.tobytes()
    assert not o.any()


@pytest.mark.parametrize("damage,msg", [
    (lambda b: b[:10], "store: truncated file"),
    (lambda b: b"HPSX" + b[4:], "store: bad magic in"),
    (lambda b: b[:4] + b"\x02\x00" + b[6:], "store: bad version in"),
    (lambda b: b[:-1], "store: size mismatch in"),
    (lambda b: b[:20] + bytes([b[20] ^ 1]) + b[21:], "store: checksum mismatch in"),
])
def test_reader_rejects_damaged_files(pkg, tmp_path, damage, msg):
    keys, emb, _ = records(50, 4, seed=2, opt=False)
    pkg.hps.write_param_files(str(tmp_path), keys, emb)
    p = tmp_path / "pf_0.bin"
    p.write_bytes(damage(p.read_bytes()))
    with pytest.raises(pkg.Error) as ei:
        pkg.hps.read_param_file(str(p))
    assert ei.value.code == "HPS_ERR_CORRUPT" and msg in str(ei.value)


def test_reader_width_mismatch(pkg, tmp_path):
    keys, emb, _ = records(10, 4, seed=4, opt=False)
    pkg.hps.write_param_files(str(tmp_path), keys, emb)
    with pytest.raises(pkg.Error, match="store: embedding width mismatch in"):
        pkg.hps.read_param_file(str(tmp_path / "pf_0.bin"), width=8)


def test_writer_argument_errors(pkg, tmp_path):
    keys, emb, _ = records(10, 4, seed=6, opt=False)
    with pytest.raises(pkg.Error, match=r"store: file_capacity must be in \[1, 65535\]"):
        pkg.hps.write_param_files(str(tmp_path), keys, emb, file_capacity=0)
    with pytest.raises(pkg.Error, match=r"store: file_capacity must be in \[1, 65535\]"):
        pkg.hps.write_param_files(str(tmp_path), keys, emb, file_capacity=65536)
    with pytest.raises(pkg.Error, match="store: dump of empty parameter set"):
        pkg.hps.write_param_files(str(tmp_path), keys[:0], emb[:0])
    with pytest.raises(pkg.Error, match="not strictly ascending"):
        pkg.hps.write_param_files(str(tmp_path), keys[::-1], emb)
    with pytest.raises(pkg.Error, match="not strictly ascending"):
        pkg.hps.write_param_files(str(tmp_path), np.r_[keys[:1], keys[:1]], emb[:2])
    assert files_of(tmp_path) == []
