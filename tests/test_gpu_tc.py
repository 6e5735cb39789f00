"""GPU: the tensor-core contraction primitive (tcgen05.mma kind::i8, Ozaki split into 7 int8
slices, 39 slice pairs in 9 exact int32 TMEM accumulators, TMA-fed A tiles) against an
extended-precision product.  Checks the value (fp64-grade) and that the rigorous per-element
bound really bounds the error."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def _exact(A, B):
    return (A.astype(np.longdouble) @ B.astype(np.longdouble).T)


@pytest.mark.parametrize("M,N,K,seed", [(128, 8, 32, 0), (200, 48, 256, 1), (90, 32, 90, 2), (256, 24, 256, 3),
                                        (37, 16, 7, 4)])
def test_ozaki_gemm_value_and_bound(M, N, K, seed):
    from paper_2605_25346_b200 import default_context
    rng = np.random.default_rng(seed)
    A = rng.normal(size=(M, K)) * np.exp(rng.uniform(-6, 6, size=(M, 1)))
    A[rng.random(A.shape) < 0.2] = 0.0
    B = rng.normal(size=(N, K)) * np.exp(rng.uniform(-3, 3, size=(N, K)))
    B[0, :] = 0.0  # a zero row
    D, E = default_context().ozaki_gemm(A, B)
    ex = _exact(A, B)
    err = np.abs(D.astype(np.longdouble) - ex)
    mag = np.abs(A) @ np.abs(B).T
    assert np.all(err <= E.astype(np.longdouble) * (1 + 1e-12) + 1e-300), float(np.max(err - E))
    # fp64-grade: bound and error both ~1e-13 of |A||B| or better
    nz = mag > 0
    assert np.all(E[~nz] == 0.0) and np.all(D[~nz] == 0.0)
    assert float(np.max(E[nz] / mag[nz])) < 1e-9
    assert float(np.max(err[nz] / mag[nz])) < 1e-11  # wide dynamic range within rows: error ~ 2^-48 of the row maxima
    assert np.all(D[:, 0] == 0.0)


@pytest.mark.parametrize("N", [40, 56, 64])
def test_ozaki_gemm_rejects_illegal_umma_n(N):
    """N = 40 / 56 raise an illegal instruction on the tensor core at M = 128 (tools/tc_shape_probe.py);
    the entry point refuses them (and N > 48, which overflows the 512 TMEM columns) up front."""
    from paper_2605_25346_b200 import default_context
    with pytest.raises(ValueError):
        default_context().ozaki_gemm(np.ones((128, 32)), np.ones((N, 32)))
