"""The seeded input generator (synth/): RNG, draw order and recipe structure."""
import numpy as np

import synth


def _splitmix64(seed: int, n: int):
    out, s = [], seed
    for _ in range(n):
        s = (s + 0x9E3779B97F4A7C15) & (2 ** 64 - 1)
        z = s
        z = ((z ^ (z >> 30)) * 0xBF58476D1CE4E5B9) & (2 ** 64 - 1)
        z = ((z ^ (z >> 27)) * 0x94D049BB133111EB) & (2 ** 64 - 1)
        out.append(z ^ (z >> 31))
    return out


def test_splitmix64_stream():
    # published first output of SplitMix64 with seed 0 (Steele, Lea, Flood 2014 reference code)
    assert _splitmix64(0, 1)[0] == 0xE220A8397B1DCDAF
    for seed in (0, 1, 1000):
        ref = _splitmix64(seed, 5)
        for k in range(5):
            assert synth.uniform_at(seed, k) == (ref[k] >> 11) * 2.0 ** -53


def test_deterministic_and_clipped():
    r = synth.resized(synth.CONFIGS["cfg3"], 96, 80).recipe
    a, b = synth.generate(r), synth.generate(r)
    assert a.dtype == np.float32 and a.shape == (1, 96, 80, 3)
    assert np.array_equal(a, b)
    assert a.min() >= 0.0 and a.max() <= 1.0


def test_quadrants_structure():
    r = synth.Recipe(1, 64, 64, 3, kind=0, noise_sigma=0.0, seed=0)
    a = synth.generate(r)[0]
    quads = [a[:32, :32], a[:32, 32:], a[32:, :32], a[32:, 32:]]  # BL, BR, TL, TR (row 0 = bottom)
    for q in quads:
        assert np.all(q == q[0, 0])
    u = [synth.uniform_at(0, k) for k in range(12)]
    for n, q in enumerate(quads):
        assert np.allclose(q[0, 0], np.float32(u[3 * n:3 * n + 3]))


def test_voronoi_cell_count_and_salt_pepper():
    r = synth.Recipe(1, 200, 160, 3, kind=1, n_cells=16, noise_sigma=0.0, seed=5)
    a = synth.generate(r)[0]
    assert len(np.unique(a.reshape(-1, 3), axis=0)) <= 16
    r2 = synth.Recipe(1, 300, 300, 3, kind=1, n_cells=8, noise_sigma=0.1, salt_pepper=0.01, seed=2)
    b = synth.generate(r2)[0]
    sp = np.mean(np.all(b == 0, -1) | np.all(b == 1, -1))
    assert 0.007 < sp < 0.014


def test_batch_seeds_independent():
    r = synth.resized(synth.CONFIGS["cfg5"], 32, 24, batch=3).recipe
    a = synth.generate(r)
    assert a.shape == (3, 32, 24, 16)
    one = synth.generate(synth.Recipe(1, 32, 24, 16, kind=1, n_cells=32, noise_sigma=0.05, seed=1001))
    assert np.array_equal(a[1], one[0])
