"""Observation files on the host: the reference's text format (io.hpp:93-131)
against a Python restatement of read_observations / write_observations, the binary format, and
the reference's error messages.  No GPU needed (the library loads, no device calls)."""
import time

import numpy as np
import pytest


@pytest.fixture(scope="module")
def cp():
    import paper_2603_25691_b200 as cp
    from paper_2603_25691_b200 import _capi
    _capi.load()
    return cp


def ref_write(path, shape, idx, vals):
    """write_observations (io.hpp:97-107): `shape:` header, 1-based indices, precision 17."""
    with open(path, "w") as f:
        f.write("shape:" + "".join(f" {n}" for n in shape) + "\n")
        for l in range(vals.size):
            f.write("".join(f"{int(idx[m, l]) + 1} " for m in range(len(shape))) + "%.17g\n" % vals[l])


def ref_read(path):
    """read_observations (io.hpp:110-131)."""
    with open(path) as f:
        lines = f.read().split("\n")
    head = lines[0].split()
    assert head[0] == "shape:"
    shape = [int(t) for t in head[1:]]
    d = len(shape)
    idx, vals = [], []
    for line in lines[1:]:
        if not line:
            continue
        tok = line.split()
        idx.append([int(t) - 1 for t in tok[:d]])
        vals.append(float(tok[d]))
    return shape, np.array(idx, dtype=np.int64).T.reshape(d, -1), np.array(vals)


def _random(cp, shape, q, seed):
    g = np.random.default_rng(seed)
    lin = g.choice(int(np.prod(shape)), size=q, replace=False)
    idx = np.array(np.unravel_index(lin, shape, order="F"), dtype=np.int64)
    vals = g.normal(size=q) * 10.0 ** g.integers(-300, 300, size=q)
    return idx, vals


@pytest.mark.parametrize("shape,q", [([7, 5, 3], 60), ([40, 30, 20, 5], 5000), ([1000], 999), ([200, 100, 100], 20000)])
def test_text_round_trip_matches_reference(cp, tmp_path, shape, q):
    idx, vals = _random(cp, shape, q, q)
    obs = cp.ObservationSet(shape, idx, vals)
    ours, ref = tmp_path / "ours.txt", tmp_path / "ref.txt"
    cp.write_observations(str(ours), obs)
    ref_write(str(ref), shape, idx, vals)
    assert ours.read_bytes() == ref.read_bytes()  # same bytes as the reference writer
    back = cp.read_observations(str(ref))
    s2, i2, v2 = ref_read(str(ref))
    assert back.shape() == shape == s2
    assert np.array_equal(back.index_array(), i2) and np.array_equal(back.index_array(), idx)
    assert np.array_equal(back.values(), v2) and np.array_equal(back.values(), vals)  # %.17g round-trips


def test_binary_round_trip(cp, tmp_path):
    shape = [64, 33, 17]
    idx, vals = _random(cp, shape, 3000, 1)
    obs = cp.ObservationSet(shape, idx, vals)
    p = tmp_path / "o.cpb"
    cp.write_observations(str(p), obs, binary=True)
    assert p.read_bytes().startswith(b"shape: 64 33 17\ncphifi-obs-binary 1 q 3000\n")
    back = cp.read_observations(str(p))
    assert back.shape() == shape
    assert np.array_equal(back.index_array(), idx) and np.array_equal(back.values(), vals)
    empty = cp.ObservationSet([3, 4], np.zeros((2, 0)), np.zeros(0), multiset=True)
    cp.write_observations(str(tmp_path / "e.cpb"), empty, binary=True)
    assert cp.read_observations(str(tmp_path / "e.cpb"), multiset=True).num_obs() == 0


def test_text_tolerances_of_the_reference_parser(cp, tmp_path):
    # blank lines skipped, tokens after the value ignored, CRLF, tabs, explicit '+' signs
    p = tmp_path / "t.txt"
    p.write_bytes(b"shape: 3 2\n\n1 1 0.5\r\n\t2 2   -1e-3 trailing tokens\n\n+3 +1 +2.25\n")
    o = cp.read_observations(str(p))
    assert o.shape() == [3, 2]
    assert np.array_equal(o.index_array(), [[0, 1, 2], [0, 1, 0]])
    assert np.array_equal(o.values(), [0.5, -1e-3, 2.25])


@pytest.mark.parametrize("content,kind,msg", [
    (b"", "runtime", "read_observations: missing shape header"),
    (b"dims: 3 3\n1 1 1.0\n", "runtime", "read_observations: expected 'shape:' header, got 'dims: 3 3'"),
    (b"shape:\n1 1.0\n", "runtime", "read_observations: empty shape header"),
    (b"shape: 3 3\n1 1 1.0\n2 2\n", "runtime", "read_observations: malformed line '2 2'"),
    (b"shape: 3 3\n1 x 1.0\n", "runtime", "read_observations: malformed line '1 x 1.0'"),
    (b"shape: 3 3\n4 1 1.0\n", "invalid", "index out of range"),
    (b"shape: 3 3\n0 1 1.0\n", "invalid", "index out of range"),
])
def test_reference_error_messages(cp, tmp_path, content, kind, msg):
    p = tmp_path / "bad.txt"
    p.write_bytes(content)
    exc = cp.CphifiRuntimeError if kind == "runtime" else cp.CphifiInvalidArgument
    with pytest.raises(exc, match=msg.replace("(", r"\(").replace(")", r"\)")):
        cp.read_observations(str(p))
    with pytest.raises(cp.CphifiRuntimeError, match="cannot open"):
        cp.read_observations(str(tmp_path / "missing.txt"))


def test_parallel_parse_throughput(cp, tmp_path):
    """2e6 records (config-1 scale x 10): the multi-threaded parser and the binary load."""
    shape = [2000, 100, 100]
    idx, vals = _random(cp, shape, 2_000_000, 7)
    obs = cp.ObservationSet(shape, idx, vals, multiset=True)
    t, b = tmp_path / "big.txt", tmp_path / "big.cpb"
    cp.write_observations(str(t), obs)
    cp.write_observations(str(b), obs, binary=True)
    t0 = time.perf_counter()
    ot = cp.read_observations(str(t), multiset=True)
    t_text = time.perf_counter() - t0
    t0 = time.perf_counter()
    ob = cp.read_observations(str(b), multiset=True)
    t_bin = time.perf_counter() - t0
    assert np.array_equal(ot.index_array(), ob.index_array()) and np.array_equal(ot.values(), ob.values())
    assert np.array_equal(ob.values(), vals)
    print(f"text parse {2e6 / t_text / 1e6:.1f} M records/s, binary {2e6 / t_bin / 1e6:.1f} M records/s")
    assert t_text < 30.0
