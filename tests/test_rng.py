"""The device random stream (DeviceRNG): Philox4x32-10 + Box-Muller + Marsaglia-Tsang.

With a DeviceRNG the step draws its StepRandoms block (sampler.py:244-260:
move_u (m,5), accept_u (m), leaf_z (m,2^D), one chi-square(nu+n)) on the
device instead of from numpy's Generator (regression.py:184).  The stream is
not numpy's, so parity runs inject the reference's blocks; these tests pin the
device stream itself:

* the bijection against known answers: Random123's philox4x32_10 vectors and
  256 vectors from PyTorch's independent CPU Philox engine
  (tests/golden/make_philox_kat.py -> philox_kat.npz);
* the block layout: each uniform is the documented 53-bit function of one
  Philox output keyed by (seed, iteration, tree, lane) -- recomputed here
  bit for bit -- and each normal is Box-Muller of one such pair;
* the distributions: KS tests of >= 1e6 device uniforms and normals, lag
  correlations, and the chi-square draw against scipy's chi2(nu+n).
"""

import os

import numpy as np
import pytest

HERE = os.path.dirname(os.path.abspath(__file__))
M0, M1, W0, W1 = 0xD2511F53, 0xCD9E8D57, 0x9E3779B9, 0xBB67AE85


def philox_np(ctr, key):
    """Random123 philox4x32_10, vectorised (ctr (k,4), key (k,2) uint32)."""
    c = np.array(ctr, np.uint64).reshape(-1, 4)
    k = np.array(key, np.uint64).reshape(-1, 2)
    mask = np.uint64(0xFFFFFFFF)
    for _ in range(10):
        p0 = c[:, 0] * np.uint64(M0)
        p1 = c[:, 2] * np.uint64(M1)
        hi0, lo0 = p0 >> np.uint64(32), p0 & mask
        hi1, lo1 = p1 >> np.uint64(32), p1 & mask
        c = np.stack([hi1 ^ c[:, 1] ^ k[:, 0], lo1, hi0 ^ c[:, 3] ^ k[:, 1], lo0], axis=1)
        k = np.stack([(k[:, 0] + np.uint64(W0)) & mask, (k[:, 1] + np.uint64(W1)) & mask], axis=1)
    return c.astype(np.uint32)


def u53(a, b):
    a = np.asarray(a, np.uint64)
    b = np.asarray(b, np.uint64)
    return ((a >> np.uint64(5)) << np.uint64(26) | (b >> np.uint64(6))).astype(np.float64) * 2.0 ** -53


def test_host_philox_matches_known_answers():
    kat = np.load(os.path.join(HERE, "golden", "philox_kat.npz"))
    np.testing.assert_array_equal(philox_np(kat["ctr"], kat["key"]), kat["out"])


def host_block(seed, it, m, size):
    """The documented device block of iteration `it` (propose.cuh propose_tree)."""
    key = np.array([seed & 0xFFFFFFFF, seed >> 32], np.uint32)
    j = np.arange(m)
    ctr = np.stack([np.full(m, it & 0xFFFFFFFF), np.full(m, it >> 32), j, np.zeros(m)], 1).astype(np.uint32)
    lanes = []
    for lane in range(3):
        ctr[:, 3] = lane
        r = philox_np(ctr, np.tile(key, (m, 1)))
        lanes.append((u53(r[:, 0], r[:, 1]), u53(r[:, 2], r[:, 3])))
    move = np.stack([lanes[0][0], lanes[0][1], lanes[1][0], lanes[1][1], lanes[2][0]], 1)
    acc = lanes[2][1]
    z = np.empty((m, size))
    for q in range((size + 1) // 2):
        ctr[:, 3] = 16 + q
        r = philox_np(ctr, np.tile(key, (m, 1)))
        u1, u2 = 1.0 - u53(r[:, 0], r[:, 1]), u53(r[:, 2], r[:, 3])
        rad = np.sqrt(-2.0 * np.log(u1))
        z[:, 2 * q] = rad * np.cos(2 * np.pi * u2)
        if 2 * q + 1 < size:
            z[:, 2 * q + 1] = rad * np.sin(2 * np.pi * u2)
    return move, acc, z


def _chain(n, p, m, D, seed):
    from paper_2410_23244_b200.sampler import DeviceRNG, Hyperparams, init_state
    rng = np.random.default_rng(seed)
    X = rng.integers(0, 16, (n, p)).astype(np.uint8)
    y = rng.normal(size=n).astype(np.float32)
    hp = Hyperparams(leaf_sd=0.3, lam=0.1, n_trees=m, max_depth=D)
    return init_state(X, np.full(p, 15), y, hp, DeviceRNG(seed), sigma2=1.0), hp


@pytest.mark.gpu
def test_device_philox_known_answers():
    from paper_2410_23244_b200.sampler import philox4x32_10
    kat = np.load(os.path.join(HERE, "golden", "philox_kat.npz"))
    np.testing.assert_array_equal(philox4x32_10(kat["ctr"], kat["key"]), kat["out"])


@pytest.mark.gpu
def test_device_block_is_the_documented_function_of_philox():
    from paper_2410_23244_b200.sampler import run
    seed = (7 << 32) | 12345
    st, hp = _chain(500, 3, 40, 6, seed)
    for _ in range(3):
        run(st, hp, 1)
        it = st.iteration - 1
        rnd = st.last_randoms()
        move, acc, z = host_block(seed, it, hp.n_trees, 1 << hp.max_depth)
        np.testing.assert_array_equal(rnd.move_u, move)  # bit-exact: integer -> u53
        np.testing.assert_array_equal(rnd.accept_u, acc)
        np.testing.assert_allclose(rnd.leaf_z, z, rtol=1e-13, atol=1e-13)  # device log/sincospi vs numpy
    st.close()


@pytest.mark.gpu
def test_device_uniforms_and_normals_distribution():
    from scipy import stats
    from paper_2410_23244_b200.sampler import run
    st, hp = _chain(300, 3, 200, 7, 99)  # 200 trees x 128 normals per step
    us, zs = [], []
    for _ in range(40):
        run(st, hp, 1)
        rnd = st.last_randoms()
        us.append(np.concatenate([rnd.move_u.ravel(), rnd.accept_u]))
        zs.append(rnd.leaf_z.ravel())
    st.close()
    u = np.concatenate(us)
    z = np.concatenate(zs)
    assert z.size >= 1_000_000
    assert u.min() >= 0.0 and u.max() < 1.0
    assert stats.kstest(u, "uniform").pvalue > 1e-3
    assert stats.kstest(z, "norm").pvalue > 1e-3
    assert abs(z.mean()) < 5 / np.sqrt(z.size) and abs(z.var() - 1) < 5 * np.sqrt(2 / z.size)
    for lag in (1, 2, 64, 128):  # within and across trees and steps
        assert abs(np.corrcoef(z[:-lag], z[lag:])[0, 1]) < 5 / np.sqrt(z.size)
    assert abs(np.corrcoef(u[:-1], u[1:])[0, 1]) < 5 / np.sqrt(u.size)


@pytest.mark.gpu
def test_device_chi_square_draw_distribution():
    """chi2(nu + n) by Marsaglia-Tsang (propose.cuh chi2_draw), as
    rng.chisquare(hp.nu + n) in the reference's block (sampler.py:259)."""
    from scipy import stats
    from paper_2410_23244_b200.sampler import run
    n = 40
    st, hp = _chain(n, 2, 1, 2, 5)
    df = hp.nu + n
    draws = []
    for _ in range(3000):
        run(st, hp, 1)
        draws.append(st.last_randoms().chi2_value)
    st.close()
    x = np.array(draws)
    assert stats.kstest(x, stats.chi2(df).cdf).pvalue > 1e-3
    assert abs(x.mean() - df) < 5 * np.sqrt(2 * df / x.size)
    assert abs(x.var() / (2 * df) - 1) < 0.15
