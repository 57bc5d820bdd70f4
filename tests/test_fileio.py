"""S24C / S24M file formats against bytes and error messages written by the
reference itself (tests/golden/formats.npz, oracle/make_golden.py)."""

from pathlib import Path

import numpy as np
import pytest
import torch

from paper_2503_16672_b200 import fileio as F
from paper_2503_16672_b200.errors import FormatError

G = np.load(Path(__file__).parent / "golden" / "formats.npz")


@pytest.mark.parametrize("tag,orient", [("tok", "token"), ("feat", "feature"), ("odd", "token")])
def test_sparse_bytes_match_reference(tag, orient):
    values, meta = G[f"{tag}_values"], G[f"{tag}_meta"]
    rows, cols = G[f"{tag}_a"].shape
    blob = F.encode_sparse(F.TOKEN_WISE if orient == "token" else F.FEATURE_WISE, rows, cols, values, meta)
    assert blob == G[f"{tag}_bytes"].tobytes()
    o, r, c, v, m = F.decode_sparse(blob)
    assert (r, c) == (rows, cols) and np.array_equal(v, values) and np.array_equal(m, meta)


def test_matrix_bytes_match_reference(tmp_path):
    a = G["mat_a"]
    assert F.encode_matrix(a) == G["mat_bytes"].tobytes()
    F.write_matrix(tmp_path / "m.s24m", a)
    assert np.array_equal(F.read_matrix(tmp_path / "m.s24m"), a)
    F.write_matrix(tmp_path / "t.s24m", torch.from_numpy(a))
    assert (tmp_path / "t.s24m").read_bytes() == G["mat_bytes"].tobytes()


@pytest.mark.parametrize("k", ["magic", "short", "trunc", "version", "orient", "m_magic", "m_trunc", "m_trail",
                               "m_nan"])
def test_malformed_files_raise_the_reference_error(k):
    blob = G[f"bad_{k}_bytes"].tobytes()
    expected = str(G[f"bad_{k}_error"])
    with pytest.raises(FormatError) as e:
        (F.decode_matrix if k.startswith("m_") else F.decode_sparse)(blob)
    assert str(e.value) == expected


@pytest.mark.gpu
def test_device_matrices_round_trip_through_s24c(tmp_path):
    """write_sparse of device sparsifications equals the oracle's bytes;
    read_sparse rebuilds values, positions and the tcgen05 metadata."""
    import paper_2503_16672_b200 as s24
    from oracle import srelu24_np as O

    rng = np.random.Generator(np.random.PCG64(55))
    a = O.bf16_round(((rng.random((256, 128)) < 0.4) * rng.standard_normal((256, 128))).astype(np.float32))
    s, _, _ = s24.sparsify_token_wise(a)
    F.write_sparse(tmp_path / "t.s24c", s)
    ov, om, _, _ = O.sparsify_token(a)
    assert (tmp_path / "t.s24c").read_bytes() == F.encode_sparse(F.TOKEN_WISE, 256, 128, ov, om)
    back = F.read_sparse(tmp_path / "t.s24c")
    assert torch.equal(back.data[:256], s.data[:256]) and torch.equal(back.meta_hw, s.meta_hw)
    f, _, _ = s24.sparsify_feature_wise(a)
    F.write_sparse(tmp_path / "f.s24c", f)
    fv, fm, _, _ = O.sparsify_feature(a)
    assert (tmp_path / "f.s24c").read_bytes() == F.encode_sparse(F.FEATURE_WISE, 256, 128, fv, fm)
    fb = F.read_sparse(tmp_path / "f.s24c")
    assert torch.equal(fb.data[:128], f.data[:128]) and torch.equal(fb.meta_hw, f.meta_hw)
