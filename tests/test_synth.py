"""The seeded input generators (synth/, shared by the oracle and the CUDA path; no method
arithmetic): structure checks of the irregular-matrix recipe the GPU sweeps use."""
import numpy as np

import synth


def _dense(A):
    return synth.csr_to_dense(A)


def test_irregular_sym_csr_structure():
    rng = np.random.default_rng(3)
    A = synth.irregular_sym_csr(400, rng, hubs=2, empty_rows=2)
    D = _dense(A)
    assert A.n == 400 and A.indptr[0] == 0 and A.indptr[-1] == len(A.indices) == len(A.data)
    np.testing.assert_array_equal(D, D.T)                          # symmetric, bitwise
    rl = np.diff(A.indptr)
    assert (rl == 0).sum() == 2                                    # the empty rows (and columns)
    for e in np.where(rl == 0)[0]:
        assert not D[:, e].any()
    assert rl.max() >= 30                                          # a hub row, longer than any gather batch (<= 8 entries)
    for i in range(A.n):                                           # sorted, unique column indices; no stored zeros
        c = A.indices[A.indptr[i]:A.indptr[i + 1]]
        assert np.all(np.diff(c) > 0)
    assert np.all(A.data != 0.0)
    ev = np.linalg.eigvalsh(D)
    assert ev[0] < -0.5 and ev[-1] > 0.5                           # indefinite


def test_irregular_sym_csr_is_seeded():
    A1 = synth.irregular_sym_csr(300, np.random.default_rng(11), hubs=1, empty_rows=0)
    A2 = synth.irregular_sym_csr(300, np.random.default_rng(11), hubs=1, empty_rows=0)
    A3 = synth.irregular_sym_csr(300, np.random.default_rng(12), hubs=1, empty_rows=0)
    assert np.array_equal(A1.indptr, A2.indptr) and np.array_equal(A1.indices, A2.indices)
    assert np.array_equal(A1.data, A2.data)
    assert not (len(A1.data) == len(A3.data) and np.array_equal(A1.data, A3.data))
