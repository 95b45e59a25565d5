"""Oracle PCG32 / stream seeding vs the reference's known answers
(proj/tests/test_rng_and_pool.cpp)."""
import numpy as np


def test_pcg32_reference_sequence(oracle):
    # test_rng_and_pool.cpp:25-31 — canonical pcg32 demo seeding (42, 54)
    r = oracle.pcg32(42, 54)
    assert [oracle.next_u32(r) for _ in range(3)] == [0xA15C02B7, 0x7B47F409, 0xBA1D3330]


def test_streams_reproducible_and_distinct(oracle):
    # test_rng_and_pool.cpp:33-45
    a, b, c = oracle.make_stream(7, 0), oracle.make_stream(7, 0), oracle.make_stream(7, 1)
    va = [oracle.next_u32(a) for _ in range(64)]
    vb = [oracle.next_u32(b) for _ in range(64)]
    vc = [oracle.next_u32(c) for _ in range(64)]
    assert va == vb
    assert not any(x == y for x, y in zip(va, vc))


def test_uniform_and_normal_moments(oracle):
    # test_rng_and_pool.cpp:47-60 (200k draws, relative tolerances 1% / 2% / 2%)
    r = oracle.make_stream(123, 9)
    n = 200000
    u = np.empty(n)
    z = np.empty(n)
    for i in range(n):
        u[i] = oracle.uniform(r, 0.0, 1.0)
        z[i] = oracle.normal(r)
    assert abs(u.mean() - 0.5) < 0.01 * 0.5
    assert abs(z.mean()) < 0.02
    assert abs((z * z).mean() - 1.0) < 0.02


def test_fill_uniform_actions_is_the_serial_stream(oracle):
    # bench.cpp:31-35: row-major fill from one stream = draw #(i*A + d)
    r1, r2 = oracle.make_stream(5, 0xAC7104), oracle.make_stream(5, 0xAC7104)
    a = oracle.fill_uniform_actions(r1, 9, 7)
    flat = [oracle.uniform(r2, -1.0, 1.0) for _ in range(63)]
    assert np.array_equal(a.reshape(-1), np.array(flat))
    assert a.min() >= -1.0 and a.max() < 1.0


def test_splitmix_stream_seeding_known_values(oracle):
    # make_stream(seed, id) = Pcg32(splitmix64(x), splitmix64(x)), x = seed ^ (K * (id + 1))
    # (rng.hpp:69-83), restated independently in Python
    M = (1 << 64) - 1

    def splitmix(x):
        x = (x + 0x9E3779B97F4A7C15) & M
        z = x
        z = ((z ^ (z >> 30)) * 0xBF58476D1CE4E5B9) & M
        z = ((z ^ (z >> 27)) * 0x94D049BB133111EB) & M
        return x, z ^ (z >> 31)

    def pcg_seed(initstate, initseq):
        inc = ((initseq << 1) | 1) & M
        s = (0 * 6364136223846793005 + inc) & M
        s = (s + initstate) & M
        s = (s * 6364136223846793005 + inc) & M
        return s, inc

    for seed, sid in [(0, 0), (0, 0xAC7104), (2024, 11), (123456789, 1 << 32)]:
        x = (seed ^ ((0x2545F4914F6CDD1D * (sid + 1)) & M)) & M
        x, a = splitmix(x)
        x, b = splitmix(x)
        s, inc = pcg_seed(a, b)
        r = oracle.make_stream(seed, sid)
        assert (r.state, r.inc) == (s, inc)
