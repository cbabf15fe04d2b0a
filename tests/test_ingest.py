"""LGT1 / JSON-lines ingest through the C ABI
(csrc/ingest.cpp): the SPEC's examples, error offsets, bit-exact round trips.
Host-only: runs without a GPU."""
import struct

import numpy as np
import pytest

import paper_2509_08383_b200 as pam


def _lgt1_bytes(vectors, version=1):
    a = np.asarray(vectors, dtype="<f4")
    return b"LGT1" + struct.pack("<HII", version, a.shape[0], a.shape[1]) + a.tobytes()


def test_minimal_lgt1(tmp_path):
    # count=1, n=2, floats [1.0, 2.0] -> one vector [1, 2]
    p = tmp_path / "min.lgt1"
    p.write_bytes(_lgt1_bytes([[1.0, 2.0]]))
    v = pam.ingest(str(p))
    assert v.dtype == np.float32 and v.shape == (1, 2) and v.tolist() == [[1.0, 2.0]]


def test_roundtrip_bit_exact(tmp_path):
    rng = np.random.default_rng(3)
    x = rng.normal(0, 3, (17, 1031)).astype(np.float32)
    x[2, 5] = np.float32(-0.0)
    x[3, 7] = np.float32(1e-45)  # subnormal
    p = tmp_path / "rt.lgt1"
    pam.write_lgt1(str(p), x)
    assert p.read_bytes() == _lgt1_bytes(x)  # little-endian, exact layout
    y = pam.ingest(str(p))
    assert y.tobytes() == x.tobytes()  # bit-exact round trip


@pytest.mark.parametrize("cut", [3, 10, 14 + 4 * 5 - 1])
def test_truncated_is_format_error(tmp_path, cut):
    b = _lgt1_bytes(np.ones((2, 3)))
    p = tmp_path / "t.lgt1"
    p.write_bytes(b[:cut])
    with pytest.raises(pam.FormatError) as e:
        pam.ingest(str(p))
    assert e.value.byte_offset >= 0


def test_bad_magic_version_trailing(tmp_path):
    p = tmp_path / "b.lgt1"
    b = bytearray(_lgt1_bytes(np.ones((1, 2))))
    b[3:4] = b"2"  # "LGT2": magic mismatch at byte 3 (a file starting with "LGT" is not JSON)
    p.write_bytes(bytes(b))
    with pytest.raises(pam.FormatError) as e:
        pam.ingest(str(p))
    assert e.value.byte_offset == 3
    p.write_bytes(_lgt1_bytes(np.ones((1, 2)), version=2))
    with pytest.raises(pam.FormatError) as e:
        pam.ingest(str(p))
    assert e.value.byte_offset == 4
    p.write_bytes(_lgt1_bytes(np.ones((1, 2))) + b"\0")
    with pytest.raises(pam.FormatError) as e:
        pam.ingest(str(p))
    assert e.value.byte_offset == 14 + 8


def test_non_finite_reports_vector(tmp_path):
    x = np.ones((4, 3), dtype=np.float32)
    x[2, 1] = np.nan
    p = tmp_path / "nf.lgt1"
    pam.write_lgt1(str(p), x)
    with pytest.raises(pam.NonFiniteError) as e:
        pam.ingest(str(p))
    assert e.value.vector_index == 2


def test_jsonl(tmp_path):
    p = tmp_path / "v.jsonl"
    p.write_text("[0.5, -0.5]\n[1e3,  2.25]\n")  # SPEC.md:551 plus a second line
    v = pam.ingest(str(p))
    assert v.dtype == np.float64 and v.tolist() == [[0.5, -0.5], [1000.0, 2.25]]
    p.write_text("[0.5, -0.5]\n[1.0]\n")  # ragged
    with pytest.raises(pam.FormatError):
        pam.ingest(str(p))
    p.write_text("[0.5, x]\n")
    with pytest.raises(pam.FormatError) as e:
        pam.ingest(str(p))
    assert e.value.byte_offset == 6
    p.write_text("[1e999, 0]\n")  # overflows to inf -> NonFinite, vector 0
    with pytest.raises(pam.NonFiniteError) as e:
        pam.ingest(str(p))
    assert e.value.vector_index == 0


@pytest.mark.gpu
def test_ingest_pinned(tmp_path):
    """SPEC.md:543-551 ingest -> pinned host tensor -> one async H2D -> the batched kernel."""
    torch = pytest.importorskip("torch")
    x = np.arange(12, dtype=np.float32).reshape(3, 4)
    p = tmp_path / "p.lgt1"
    pam.write_lgt1(str(p), x)
    t = pam.ingest_pinned(str(p))
    assert t.is_pinned() and t.numpy().tobytes() == x.tobytes()
    # the pinned upload feeds the fp32 batch entry point
    rng = np.random.default_rng(3)
    big = rng.normal(0, 3, (8, 4096)).astype(np.float32)
    pam.write_lgt1(str(p), big)
    tp = pam.ingest_pinned(str(p))
    d = tp.to("cuda", non_blocking=True)
    z, am, st = pam.cutmax_batch_device(d, pam.CutMaxParams())
    torch.cuda.synchronize()
    assert np.array_equal(am.cpu().numpy(), big.argmax(1)) and int(st.abs().sum()) == 0
