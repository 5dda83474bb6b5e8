"""On-disk index format (include/rd_format.h).

CPU tests run the oracle's save / load; the GPU tests cross the two libraries
(engine file -> oracle, oracle file -> engine) so the format is one spec, and
check that an engine index with offloaded lists saves every list."""
import os
import struct

import numpy as np
import pytest

from paper_2504_15302_b200.retriever import ParseError

HEADER = struct.Struct("<8sIIqiiQQQQQQ")


def _same_layout(a, b):
    ao, ai, _ = a.layout()
    bo, bi, _ = b.layout()
    np.testing.assert_array_equal(ao, bo)
    np.testing.assert_array_equal(ai, bi)


def test_oracle_roundtrip(oracle, tmp_path):
    desc = oracle.desc(6000, 96, 13, shard=1, num_shards=3)
    idx = oracle.synthetic_index(desc)
    path = str(tmp_path / "kb.rdidx")
    idx.save(path)
    back = oracle.load_index(path)
    _same_layout(idx, back)
    q, _ = oracle.synth_queries(desc, 0, 9)
    a, b = idx.search(q, 4, 10), back.search(q, 4, 10)
    np.testing.assert_array_equal(a.ids, b.ids)
    np.testing.assert_array_equal(a.dists, b.dists)


def test_header_layout(oracle, tmp_path):
    desc = oracle.desc(1000, 64, 7)
    path = str(tmp_path / "kb.rdidx")
    oracle.synthetic_index(desc).save(path)
    raw = open(path, "rb").read()
    magic, ver, flags, n, d, nlist, o_off, o_ids, o_c, o_v, size, _ = HEADER.unpack_from(raw, 0)
    assert magic == b"RDIDX\0v1" and ver == 1 and flags == 0
    assert (n, d, nlist) == (1000, 64, 7)
    assert all(o % 4096 == 0 for o in (o_off, o_ids, o_c, o_v))
    assert size == len(raw) == o_v + 4 * n * d
    offs = np.frombuffer(raw, dtype=np.int64, count=nlist + 1, offset=o_off)
    assert offs[0] == 0 and offs[-1] == n


def test_host_index_with_ids_roundtrip(oracle, tmp_path):
    rng = np.random.default_rng(3)
    X = rng.standard_normal((500, 32)).astype(np.float32)
    C = rng.standard_normal((4, 32)).astype(np.float32)
    offs = np.array([0, 100, 100, 350, 500], dtype=np.int64)  # includes an empty list
    ids = rng.permutation(10_000)[:500].astype(np.int64)
    idx = oracle.index_from_host(X, offs, C, ids)
    path = str(tmp_path / "h.rdidx")
    idx.save(path)
    back = oracle.load_index(path)
    _same_layout(idx, back)
    r = back.search(X[:7], 4, 3)
    np.testing.assert_array_equal(r.ids[:, 0], ids[:7])


@pytest.mark.parametrize("damage", ["magic", "truncate", "offsets", "missing", "version"])
def test_malformed_files_are_parse_errors(oracle, tmp_path, damage):
    desc = oracle.desc(800, 32, 5)
    path = str(tmp_path / "kb.rdidx")
    oracle.synthetic_index(desc).save(path)
    raw = bytearray(open(path, "rb").read())
    if damage == "magic":
        raw[0:5] = b"XXXXX"
    elif damage == "truncate":
        raw = raw[: len(raw) - 100]
    elif damage == "offsets":
        raw[4096 + 8] ^= 0x01  # list_offsets[1]: checksum no longer matches
    elif damage == "version":
        raw[8] = 9
    if damage == "missing":
        path = str(tmp_path / "absent.rdidx")
    else:
        open(path, "wb").write(bytes(raw))
    with pytest.raises(ParseError):
        oracle.load_index(path)


@pytest.mark.gpu
def test_engine_file_loads_in_oracle_and_back(engine, oracle, tmp_path):
    desc = engine.desc(30000, 768, 48)
    e = engine.synthetic_index(desc)
    o = oracle.synthetic_index(desc)
    ep, op = str(tmp_path / "e.rdidx"), str(tmp_path / "o.rdidx")
    e.save(ep)
    o.save(op)
    assert open(ep, "rb").read() == open(op, "rb").read(), "engine and oracle must write identical files"
    oe = oracle.load_index(ep)
    eo = engine.load_index(op)
    _same_layout(oe, o)
    _same_layout(eo, e)
    q, _ = engine.synth_queries(desc, 100, 40)
    want = o.search(q, 8, 10)
    for got in (eo.search(q, 8, 10), oe.search(q, 8, 10)):
        np.testing.assert_array_equal(got.ids, want.ids)
        np.testing.assert_array_equal(got.dists, want.dists)


@pytest.mark.gpu
def test_engine_saves_offloaded_lists(engine, oracle, tmp_path):
    desc = engine.desc(20000, 768, 32)
    e = engine.synthetic_index(desc)
    e.place(offload_fraction=0.5)
    assert e.info()["lists_resident"] == 16
    path = str(tmp_path / "off.rdidx")
    e.save(path)
    o = oracle.synthetic_index(desc)
    op = str(tmp_path / "o.rdidx")
    o.save(op)
    assert open(path, "rb").read() == open(op, "rb").read()
    back = engine.load_index(path)
    assert back.info()["lists_resident"] == 32
    q, _ = engine.synth_queries(desc, 5, 16)
    want = o.search(q, 6, 10)
    got = back.search(q, 6, 10)
    np.testing.assert_array_equal(got.ids, want.ids)
    np.testing.assert_array_equal(got.dists, want.dists)
