"""NEXT-4: Matrix Market ingestion (phipm_mm_read, host code) against scipy.io's independent reader
and writer: general, symmetric, skew-symmetric, pattern and integer files, duplicates, comments,
and malformed input.  CPU only."""
import io
import os

import numpy as np
import pytest
import scipy.io
import scipy.sparse as sp

import paper_0907_4631_b200 as P
import workloads as W


def roundtrip(tmp_path, A, **kw):
    p = os.path.join(tmp_path, "a.mtx")
    scipy.io.mmwrite(p, A, **kw)
    rp, col, val = P.read_matrix_market(p)
    ref = sp.csr_matrix(scipy.io.mmread(p))
    ref.sum_duplicates()
    ref.sort_indices()
    return (rp, col, val), ref


@pytest.fixture(scope="module", autouse=True)
def built():
    P.build()


def test_general_roundtrip_is_exact(tmp_path):
    rp, col, val = W.make("c5_mini").csr
    A = sp.csr_matrix((val, col, rp), shape=(len(rp) - 1,) * 2)
    (r2, c2, v2), ref = roundtrip(tmp_path, A, precision=17)
    assert np.array_equal(r2, rp) and np.array_equal(c2, col)
    assert np.array_equal(v2, val)                      # 17 significant digits: exact doubles


@pytest.mark.parametrize("kind", ["symmetric", "skew-symmetric"])
def test_symmetric_storage_expanded(tmp_path, kind):
    rng = np.random.default_rng(7)
    B = sp.random(60, 60, density=0.1, random_state=8, format="csr")
    A = (B + B.T) if kind == "symmetric" else (B - B.T)
    if kind == "symmetric":
        A = A + sp.eye(60)
    A = sp.csr_matrix(A)
    A.eliminate_zeros()
    (rp, col, val), ref = roundtrip(tmp_path, A, symmetry=kind, precision=17)
    assert np.array_equal(rp, ref.indptr) and np.array_equal(col, ref.indices)
    assert np.array_equal(val, ref.data)
    D = sp.csr_matrix((val, col, rp), shape=A.shape).toarray()
    assert np.array_equal(D, A.toarray())


def test_pattern_integer_comments(tmp_path):
    p = os.path.join(tmp_path, "b.mtx")
    open(p, "w").write("%%MatrixMarket matrix coordinate integer general\n% a comment\n\n"
                       "3 3 4\n1 1 7\n3 2 -1\n% mid comment\n2 3 4\n1 3 1\n")
    rp, col, val = P.read_matrix_market(p)
    assert rp.tolist() == [0, 2, 3, 4] and col.tolist() == [0, 2, 2, 1] and val.tolist() == [7.0, 1.0, 4.0, -1.0]
    q = os.path.join(tmp_path, "c.mtx")
    open(q, "w").write("%%MatrixMarket matrix coordinate pattern symmetric\n3 3 2\n2 1\n3 3\n")
    rp, col, val = P.read_matrix_market(q)
    assert rp.tolist() == [0, 1, 2, 3] and col.tolist() == [1, 0, 2] and val.tolist() == [1.0, 1.0, 1.0]


@pytest.mark.parametrize("text", [
    "%%MatrixMarket matrix array real general\n2 2\n1\n2\n3\n4\n",          # dense array format
    "%%MatrixMarket matrix coordinate real general\n2 3 1\n1 1 1\n",         # not square
    "%%MatrixMarket matrix coordinate real general\n2 2 1\n3 1 1\n",         # index out of range
    "%%MatrixMarket matrix coordinate complex general\n2 2 1\n1 1 1 0\n",    # complex
    "%%MatrixMarket matrix coordinate real general\n2 2 2\n1 1 1\n",         # truncated
    "not a matrix market file\n",
    "%%MatrixMarket matrix coordinate real general\n2 2 2\n1 1 1\n1 1 5\n",  # duplicate
    "%%MatrixMarket matrix coordinate real symmetric\n2 2 3\n1 1 1\n2 1 2\n1 2 2\n",  # both triangles
])
def test_rejects_malformed(tmp_path, text):
    p = os.path.join(tmp_path, "bad.mtx")
    open(p, "w").write(text)
    with pytest.raises(P.PhipmError):
        P.read_matrix_market(p)
    with pytest.raises(P.PhipmError):
        P.read_matrix_market(os.path.join(tmp_path, "missing.mtx"))
