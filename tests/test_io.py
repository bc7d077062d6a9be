"""Table files: binary ingest (read_binary,
P/src/relation.cpp:98-127), the pair writers (save_table, :164-204) and
format detection (:13-20). The CPU tests cover detection and the host-side
size checks; the GPU tests mirror P/tests/test_relation.cpp:67-105 and
P/tests/test_cli.cpp:191-210 through the C ABI."""
import os

import numpy as np
import pytest

import paper_2206_04995_b200 as d3
from support import SplitMix64, oracle_pairs, pair_set, random_instance

C = d3.CostConstants.test_consts()
F = d3.FileFormat


def _interleaved(left, right):
    out = np.empty(2 * len(left), dtype=np.uint64)
    out[0::2] = left
    out[1::2] = right
    return out


def _text(left, right, sep):
    return "".join(f"{int(a)}{sep}{int(b)}\n" for a, b in zip(left, right)).encode()


# ---- CPU -------------------------------------------------------------------
def test_detect_format_by_extension():
    """detect_format (relation.cpp:13-20): requested wins, else .tsv/.txt,
    .csv, .bin, anything else tsv."""
    assert d3.detect_format("r.tsv") == F.tsv
    assert d3.detect_format("r.txt") == F.tsv
    assert d3.detect_format("a/b/r.csv") == F.csv
    assert d3.detect_format("r.bin") == F.binary
    assert d3.detect_format("r") == F.tsv
    assert d3.detect_format("dir.bin/r") == F.tsv
    assert d3.detect_format("r.tsv", F.binary) == F.binary


def test_binary_rows_and_errors(tmp_path):
    """read_binary's checks: missing file -> IoError, length not a multiple
    of 16 -> FormatError (relation.cpp:99-106)."""
    p = tmp_path / "t.bin"
    _interleaved(np.arange(5, dtype=np.uint64), np.arange(5, dtype=np.uint64)).tofile(p)
    assert d3.binary_rows(p) == 5
    np.arange(5, dtype=np.uint64).tofile(p)  # 40 bytes
    with pytest.raises(d3.FormatError):
        d3.binary_rows(p)
    with pytest.raises(d3.IoError):
        d3.binary_rows(tmp_path / "missing.bin")
    p.write_bytes(b"")
    assert d3.binary_rows(p) == 0


# ---- GPU -------------------------------------------------------------------
@pytest.mark.gpu
def test_binary_round_trip_is_exact(tmp_path):
    """test_relation.cpp:67-78, and the bytes are the reference's layout
    (little-endian u64 left, right per row, no header)."""
    i = np.arange(1000, dtype=np.uint64)
    left = i * np.uint64(0x9E3779B97F4A7C15)
    right = ~i
    p = tmp_path / "rel_rt.bin"
    d3.save_table(d3.RawTable(left, right), p, F.binary)
    assert p.read_bytes() == _interleaved(left, right).tobytes()
    t = d3.load_table(p)
    assert t.size() == 1000
    assert np.array_equal(t.left.cpu().numpy().view(np.uint64), left)
    assert np.array_equal(t.right.cpu().numpy().view(np.uint64), right)


@pytest.mark.gpu
@pytest.mark.parametrize("fmt,sep,ext", [(F.tsv, "\t", "tsv"), (F.csv, ",", "csv")])
def test_text_writer_matches_reference_format(tmp_path, fmt, sep, ext):
    """test_relation.cpp:80-94: u64 max survives text; every line is
    "left<sep>right\\n" in decimal, byte-identical to the reference writer."""
    p = tmp_path / f"rel_rt.{ext}"
    left = np.array([18446744073709551615, 42, 0, 9, 10, 99, 100], dtype=np.uint64)
    right = np.array([0, 7, 1, 10, 9, 1000, 10**19], dtype=np.uint64)
    d3.save_table(d3.RawTable(left, right), p, fmt)
    assert p.read_bytes() == _text(left, right, sep)
    rng = np.random.default_rng(7)
    left = rng.integers(0, 2**64, 20000, dtype=np.uint64)
    right = (rng.integers(0, 2**64, 20000, dtype=np.uint64) >> rng.integers(0, 64, 20000,
                                                                         dtype=np.uint64))
    d3.save_table(d3.RawTable(left, right), p, fmt)
    assert p.read_bytes() == _text(left, right, sep)


@pytest.mark.gpu
def test_auto_format_detection(tmp_path):
    """test_relation.cpp:96-105: .bin written with auto detection is binary."""
    pb = tmp_path / "rel_auto.bin"
    d3.save_table(d3.RawTable(np.array([1], np.uint64), np.array([2], np.uint64)), pb)
    assert pb.read_bytes() == _interleaved(np.array([1], np.uint64), np.array([2], np.uint64)).tobytes()
    assert d3.load_table(pb).left.cpu().tolist() == [1]


@pytest.mark.gpu
def test_multi_chunk_files_keep_row_order(tmp_path):
    """Tables larger than the pinned chunks (64 MB read / 2M-row write) stream
    in order, device columns in, device columns out."""
    import torch
    rl, rr = d3.generate(2, 0)  # 5M rows on the device
    p = tmp_path / "big.bin"
    d3.save_table(d3.RawTable(rl, rr), p)
    want = _interleaved(rl.cpu().numpy().view(np.uint64), rr.cpu().numpy().view(np.uint64))
    assert np.array_equal(np.fromfile(p, dtype=np.uint64), want)
    t = d3.load_table(p)
    assert torch.equal(t.left, rl) and torch.equal(t.right, rr)
    pt = tmp_path / "big.tsv"
    n = 2_500_000
    d3.save_table(d3.RawTable(rl[:n].contiguous(), rr[:n].contiguous()), pt)
    got = np.loadtxt(pt, dtype=np.uint64, delimiter="\t")
    assert np.array_equal(got[:, 0], rl[:n].cpu().numpy().view(np.uint64))
    assert np.array_equal(got[:, 1], rr[:n].cpu().numpy().view(np.uint64))


@pytest.mark.gpu
def test_binary_tables_through_the_engine(tmp_path):
    """test_cli.cpp:191-210: binary-loaded (device) tables give the same
    result as the host tables, and --out writes the decoded pairs."""
    rng = SplitMix64(505)
    for k in range(5):
        r, s = random_instance(rng)
        pr, ps = tmp_path / f"r{k}.bin", tmp_path / f"s{k}.bin"
        _interleaved(*r).tofile(pr)
        _interleaved(*s).tofile(ps)
        cfg = d3.EngineConfig(force=d3.Strategy.auto_select)
        out = d3.join_project(d3.load_table(pr), d3.load_table(ps), cfg, C)
        assert pair_set(out.result.raw_x, out.result.raw_z) == oracle_pairs(r, s)
        po = tmp_path / f"out{k}.tsv"
        d3.save_result(out, po)
        raw = d3.result_to_raw(out)
        assert po.read_bytes() == _text(raw.raw_x, raw.raw_z, "\t")
