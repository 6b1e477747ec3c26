"""Input-generator pins (-m "not gpu"): the counter-based Philox4x32-10 used
for the device-generated C5 matrix reproduces the Random123 known-answer
vectors, and the C5 entries have the stated law (mean 0, variance 1/m)."""
import numpy as np

import synth
import synth.philox as ph


def test_philox_known_answers():
    f = 0xFFFFFFFF
    kat = [((0, 0, 0, 0, 0, 0), (0x6627E8D5, 0xE169C58D, 0xBC57AC4C, 0x9B00DBD8)),
           ((f, f, f, f, f, f), (0x408F276D, 0x41C83B0E, 0xA20BC7C6, 0x6D5451FD)),
           ((0x243F6A88, 0x85A308D3, 0x13198A2E, 0x03707344, 0xA4093822, 0x299F31D0),
            (0xD16CFE09, 0x94FDCCEB, 0x5001E420, 0x24126EA1))]
    for args, out in kat:
        assert tuple(int(v) for v in ph.philox4x32_10(*args)) == out


def test_c5_entry_law():
    m = 100000
    A = ph.centered_block(np.arange(2000), np.arange(50), m, seed=5)
    assert abs(A.mean()) < 4 * np.sqrt(1.0 / m / A.size)
    assert abs(A.var() * m - 1.0) < 0.02
    assert np.max(np.abs(A)) <= np.sqrt(3.0 / m) + 1e-15


def test_generators_deterministic():
    a = synth.nnls_gaussian(30, 20, 7)
    b = synth.nnls_gaussian(30, 20, 7)
    assert np.array_equal(a.M, b.M) and np.array_equal(a.b, b.b)
    assert a.M.flags.f_contiguous


def test_weak_shards_independent_of_b():
    """Regression: the weak-scaling shards must not share a random stream with b
    (numpy SeedSequence([s, 0]) == SeedSequence(s) once made column 0 of A = b/sqrt(m))."""
    p0, p1 = synth.weak_shard(300, 50, 0, 2), synth.weak_shard(300, 50, 1, 2)
    assert np.array_equal(p0.b, p1.b)
    for p in (p0, p1):
        c = np.abs(p.M.T @ p.b) / (np.linalg.norm(p.M, axis=0) * np.linalg.norm(p.b))
        assert c.max() < 0.5
    assert not np.allclose(p0.M, p1.M)
