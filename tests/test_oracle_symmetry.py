"""Symmetry pins of the whole oracle trajectory (steps 1-5 together, Δt > 0, several multiplier
rounds) - the part SURVEY §8(c) P20 leaves without a closed form. Nothing in the method
distinguishes the two image axes when h_x = h_y, nor the colour channels:
  * transpose equivariance: on a square image, the run on I^T is the transpose of the run on I
    with the two halves of p and mu exchanged ((x,k) <-> (y,k)); the window D_R, the spatial term
    |delta|_h^2, the forward-difference gradient, its adjoint divergence, the coupled pixel norm
    and the Huber / shrink steps are all invariant under the swap;
  * channel permutation equivariance: the coupled norms and the colour distance are sums over
    channels, so permuting the channels of I permutes c, cbar and each half of p, mu.
Only the summation order of the offsets (dx-major) and of the channels changes, so agreement is
to fp64 rounding. A transposed operand, a p_x / p_y mix-up in div or in the dual step, an h_x /
h_y swap (here h_x = h_y, so caught through the index pattern) or a channel-dependent constant
breaks one of these."""
import numpy as np
import pytest

import oracle

pytestmark = pytest.mark.filterwarnings("ignore")


def _run(I, scheme, kernel, R, K=3, rounds=3):
    H, W, C = I.shape
    h = 1.0 / (W - 1)
    p = oracle.Params(height=H, width=W, channels=C, radius=R, kernel=kernel, iters_per_round=K, rounds=rounds,
                      alpha=8.0 / h, beta=1.0, eps_c=20.0, dt=0.25, rho=2.5 * h, gamma=2.5 * h,
                      kappa=1.0 if scheme else 1.3, scheme=scheme)
    s = oracle.solve(p, I)
    return s, np.array(s.stats)


def _img(seed, H, W, C):
    rng = np.random.default_rng(seed)
    blocks = np.repeat(np.repeat(rng.random((3, 3, C)), (H + 2) // 3, 0)[:H], (W + 2) // 3, 1)[:, :W]
    return np.clip(blocks + 0.08 * rng.standard_normal((H, W, C)), 0, 1)


@pytest.mark.parametrize("scheme,kernel,R", [(0, 0, 2), (0, 1, 3), (1, 0, 3)])
def test_transpose_equivariance(scheme, kernel, R):
    I = _img(R + 10 * scheme, 13, 13, 3)
    a, sa = _run(I, scheme, kernel, R)
    b, sb = _run(I.transpose(1, 0, 2).copy(), scheme, kernel, R)
    C = I.shape[2]
    tol = 1e-12
    np.testing.assert_allclose(b.c, a.c.transpose(1, 0, 2), rtol=0, atol=tol)
    np.testing.assert_allclose(b.cbar, a.cbar.transpose(1, 0, 2), rtol=0, atol=tol)
    swap = np.r_[np.arange(C, 2 * C), np.arange(C)]  # (x,k) <-> (y,k)
    scale = max(1.0, float(np.max(np.abs(a.p))))
    np.testing.assert_allclose(b.p, a.p.transpose(1, 0, 2)[..., swap], rtol=0, atol=tol * scale)
    scale = max(1.0, float(np.max(np.abs(a.mu))))
    np.testing.assert_allclose(b.mu, a.mu.transpose(1, 0, 2)[..., swap], rtol=0, atol=tol * scale)
    np.testing.assert_allclose(sb, sa, rtol=1e-10, atol=1e-12)
    # the run is not trivially symmetric: the image is not, and neither is the result
    assert np.max(np.abs(a.c - a.c.transpose(1, 0, 2))) > 1e-3


@pytest.mark.parametrize("scheme,C,perm", [(0, 3, [2, 0, 1]), (1, 3, [1, 2, 0]), (0, 5, [4, 1, 3, 0, 2])])
def test_channel_permutation_equivariance(scheme, C, perm):
    I = _img(7 + C, 11, 14, C)
    a, sa = _run(I, scheme, 0, 2)
    b, sb = _run(I[..., perm].copy(), scheme, 0, 2)
    perm2 = np.r_[np.array(perm), C + np.array(perm)]
    tol = 1e-12
    np.testing.assert_allclose(b.c, a.c[..., perm], rtol=0, atol=tol)
    np.testing.assert_allclose(b.cbar, a.cbar[..., perm], rtol=0, atol=tol)
    np.testing.assert_allclose(b.p, a.p[..., perm2], rtol=0, atol=tol * max(1.0, float(np.max(np.abs(a.p)))))
    np.testing.assert_allclose(b.mu, a.mu[..., perm2], rtol=0, atol=tol * max(1.0, float(np.max(np.abs(a.mu)))))
    nf = sa.shape[1] - C  # fixed statistics, then the per-channel means
    np.testing.assert_allclose(sb[:, :nf], sa[:, :nf], rtol=1e-10, atol=1e-12)
    np.testing.assert_allclose(sb[:, nf:], sa[:, nf:][:, perm], rtol=1e-12, atol=1e-14)
