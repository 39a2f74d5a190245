"""Block-coordinate text format (reference dump_block_coo, blockla.hpp:253-268,
and its round-trip test tests/test_blockla.cpp:207-230).

CPU: the product's writer emits byte-identical text to the reference's own
dump (oracle/_ref), and the reader rebuilds the matrix bit-exactly the way
the reference's BlockBuilder does.  GPU: dump of a device BSR and upload of a
dump through the C ABI."""
import numpy as np
import pytest

import paper_2412_12506_b200 as g
from tests.cases import scalar


def _random_bsr(rng, brows, bcols, rbs, cbs, density, signed_zero=False):
    ptr, col = [0], []
    for _ in range(brows):
        js = [j for j in range(bcols) if rng.random() < density]
        col += js
        ptr.append(len(col))
    val = rng.standard_normal(len(col) * rbs * cbs)
    # values that stress %.17g: tiny, huge, exact integers, subnormals, -0
    special = [1.0, -0.0 if signed_zero else 0.0, 1e-310, 1.7976931348623157e308, 0.1, -2.5e-17, 3.0]
    val[: min(len(val), len(special))] = special[: len(val)]
    return np.array(ptr, np.int32), np.array(col, np.int32), val


@pytest.mark.parametrize("shape", [(4, 4, 2, 3), (7, 5, 3, 3), (1, 1, 1, 1), (0, 3, 2, 2)])
def test_writer_matches_reference_dump(ref, tmp_path, shape):
    rng = np.random.default_rng(37)
    brows, bcols, rbs, cbs = shape
    ptr, col, val = _random_bsr(rng, brows, bcols, rbs, cbs, 0.5)
    ours, theirs = tmp_path / "ours.txt", tmp_path / "ref.txt"
    g.coo_write(ours, brows, bcols, rbs, cbs, ptr, col, val)
    ref.dump_block_coo(brows, bcols, rbs, cbs, ptr, col, val, theirs)
    assert ours.read_bytes() == theirs.read_bytes()


def test_level_operator_dump_matches_reference(ref, tmp_path):
    P = g.Problem(scalar(8, 2, degree=2))
    n, bs, _ = P.level_shape(0)
    ptr, col, val = P.level_matrix(0)
    ours, theirs = tmp_path / "A.txt", tmp_path / "A_ref.txt"
    g.coo_write(ours, n, n, bs, bs, ptr, col, val)
    ref.dump_block_coo(n, n, bs, bs, ptr, col, val, theirs)
    assert ours.read_bytes() == theirs.read_bytes()
    assert ours.read_text().splitlines()[0] == f"blockcoo {n} {n} {bs} {bs} {len(col)}"


def test_round_trip_is_bit_exact(tmp_path):
    rng = np.random.default_rng(5)
    ptr, col, val = _random_bsr(rng, 9, 6, 2, 3, 0.6)
    path = tmp_path / "m.txt"
    g.coo_write(path, 9, 6, 2, 3, ptr, col, val)
    br, bc, rb, cb, p2, c2, v2 = g.coo_read(path)
    assert (br, bc, rb, cb) == (9, 6, 2, 3)
    assert np.array_equal(p2, ptr) and np.array_equal(c2, col)
    assert v2.tobytes() == val.tobytes()  # max_digits10 round trip is exact


def test_reader_follows_block_builder(tmp_path):
    # unordered blocks, a duplicate (summed in file order), -0.0 (0.0 + -0.0 = +0.0)
    path = tmp_path / "d.txt"
    path.write_text("blockcoo 2 3 1 2 4\n"
                    "1 2 1 2\n"
                    "0 1 -0 5\n"
                    "1 0 0.5 0.25\n"
                    "1 2 0.1 0.2\n")
    br, bc, rb, cb, ptr, col, val = g.coo_read(path)
    assert (br, bc, rb, cb) == (2, 3, 1, 2)
    assert ptr.tolist() == [0, 1, 3] and col.tolist() == [1, 0, 2]
    want = np.array([0.0 + -0.0, 0.0 + 5.0, 0.5, 0.25, (0.0 + 1.0) + 0.1, (0.0 + 2.0) + 0.2])
    assert val.tobytes() == want.tobytes()
    assert not np.signbit(val[0])


@pytest.mark.parametrize("text,err", [
    ("blockcoox 1 1 1 1 0\n", "missing header"),
    ("blockcoo 1 1 1 1 1\n0 3 1.0\n", "out of range"),
    ("blockcoo 1 1 1 1 1\n0 0\n", "truncated"),
    ("blockcoo 1 1 1 1 1\n0 0 abc\n", "bad number"),
])
def test_reader_errors(tmp_path, text, err):
    path = tmp_path / "bad.txt"
    path.write_text(text)
    with pytest.raises(g.LdgmgRuntimeError, match=err):
        g.coo_read(path)
    with pytest.raises(g.LdgmgRuntimeError, match="cannot open"):
        g.coo_read(tmp_path / "missing.txt")


@pytest.mark.gpu
def test_device_dump_and_load(ctx, tmp_path):
    rng = np.random.default_rng(11)
    ptr, col, val = _random_bsr(rng, 12, 12, 3, 3, 0.4)
    A = g.DeviceBsr(ctx, 12, 12, 3, 3, ptr, col, val)
    dev, host = tmp_path / "dev.txt", tmp_path / "host.txt"
    A.dump_coo(dev)
    g.coo_write(host, 12, 12, 3, 3, ptr, col, val)
    assert dev.read_bytes() == host.read_bytes()
    B = g.DeviceBsr.load_coo(ctx, dev)
    assert (B.brows, B.bcols, B.row_bs, B.col_bs, B.nnzb) == (12, 12, 3, 3, len(col))
    p2, c2, v2 = B.download()
    assert np.array_equal(p2, ptr) and np.array_equal(c2, col) and v2.tobytes() == val.tobytes()
