"""MMX1 loader: header validation with the reference's
messages (io.py:90-106) on CPU; streaming the payload to the device through
pinned chunks, fp64 bitwise and fp32 = numpy astype(float32), on the GPU."""

import struct

import numpy as np
import pytest

import paper_1003_3272_b200 as M
from paper_1003_3272_b200.errors import MatrixFormatError


def write_mmx(path, a):
    a = np.ascontiguousarray(a, dtype="<f8")
    with open(path, "wb") as fh:
        fh.write(b"MMX1")
        fh.write(struct.pack("<QQ", *a.shape))
        fh.write(a.tobytes(order="C"))


def test_header_round_trip(tmp_path):
    p = tmp_path / "a.mmx"
    write_mmx(p, np.zeros((3, 5)))
    assert M.read_mmx_header(p) == (3, 5)


def test_bad_magic(tmp_path):
    p = tmp_path / "a.mmx"
    p.write_bytes(b"MMX2" + struct.pack("<QQ", 1, 1) + b"\0" * 8)
    with pytest.raises(MatrixFormatError) as e:
        M.read_mmx_header(p)
    assert str(e.value) == f"{p}: bad magic b'MMX2', expected b'MMX1'"


def test_truncated_header(tmp_path):
    p = tmp_path / "a.mmx"
    p.write_bytes(b"MMX1" + b"\1\0\0")
    with pytest.raises(MatrixFormatError) as e:
        M.read_mmx_header(p)
    assert str(e.value) == f"{p}: truncated header (7 bytes)"


def test_payload_length(tmp_path):
    p = tmp_path / "a.mmx"
    p.write_bytes(b"MMX1" + struct.pack("<QQ", 2, 3) + b"\0" * 40)
    with pytest.raises(MatrixFormatError) as e:
        M.read_mmx_header(p)
    assert str(e.value) == f"{p}: payload for 2x3 needs 68 bytes, file has 60"


@pytest.mark.gpu
@pytest.mark.parametrize("dtype", ["fp32", "fp64"])
@pytest.mark.parametrize("shape,chunk", [((257, 131), 4096 + 32), ((1, 7), 32), ((0, 5), 1 << 20),
                                         ((2048, 1500), 1 << 20)])
def test_load_matrix_device(tmp_path, dtype, shape, chunk):
    rng = np.random.default_rng(7)
    a = rng.standard_normal(shape) * np.exp(rng.uniform(-30, 30, shape))
    p = tmp_path / "x.mmx"
    write_mmx(p, a)
    t = M.load_matrix_device(p, M.Backend(dtype=dtype), chunk_bytes=chunk)
    want = a.astype(np.float32) if dtype == "fp32" else a
    got = t.cpu().numpy()
    assert got.dtype == want.dtype and got.shape == want.shape
    np.testing.assert_array_equal(got.view(np.uint32 if dtype == "fp32" else np.uint64),
                                  want.view(np.uint32 if dtype == "fp32" else np.uint64))


@pytest.mark.gpu
def test_loaded_matrix_feeds_nnmf(tmp_path):
    rng = np.random.default_rng(3)
    x = rng.random((300, 64))
    p = tmp_path / "x.mmx"
    write_mmx(p, x)
    be = M.Backend(dtype="fp64")
    xd = M.load_matrix_device(p, be)
    s0 = M.FactorPair(rng.random((300, 4)), rng.random((4, 64)))
    cfg = M.MmConfig(max_iters=20, epsilon=1e-300)
    _, t_dev = M.nnmf_run(M.NnmfProblem(x=xd, rank=4), cfg, be, state0=s0)
    _, t_host = M.nnmf_run(M.NnmfProblem(x=x, rank=4), cfg, be, state0=s0)
    np.testing.assert_array_equal(t_dev.objective_values, t_host.objective_values)
