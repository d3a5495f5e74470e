"""LBFIELD checkpoint format round trip, CPU only."""
import numpy as np
import pytest

import lbgen
from paper_1703_00186_b200 import checkpoint


def test_lbfield_roundtrip(tmp_path):
    st = lbgen.random_field(37, 9, 13, seed=2)
    p = str(tmp_path / "a.lbfield")
    checkpoint.save(p, st)
    raw = open(p, "rb").read()
    assert raw.startswith(b"LBFIELD 37 9 13\n")
    assert len(raw) == len(b"LBFIELD 37 9 13\n") + 37 * 9 * 13 * 8
    back = checkpoint.load(p)
    assert back.shape == st.shape and np.array_equal(back, st)


def test_lbfield_rejects_garbage(tmp_path):
    p = tmp_path / "b.lbfield"
    p.write_bytes(b"NOTLB 1 2 3\n")
    with pytest.raises(ValueError):
        checkpoint.load(str(p))
    p.write_bytes(b"LBFIELD 37 2 2\n" + b"\0" * 8)
    with pytest.raises(ValueError):
        checkpoint.load(str(p))
