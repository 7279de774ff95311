"""The seeded input generators (synth/) -- host side; the device twin is checked in test_gpu_parity."""
import numpy as np

import synth


def test_random_access_consistent():
    big = synth.data(10000, seed=0)
    for off, n in ((0, 1), (1, 7), (7, 9), (8, 8), (13, 4000), (9991, 9)):
        assert synth.stream_bytes(0, 0, off, n).tobytes() == big[off: off + n].tobytes()


def test_known_first_word():
    # splitmix64 with key 0: first output of the reference generator (state += gamma, then mix)
    z = (0x9E3779B97F4A7C15) & (2 ** 64 - 1)
    z = ((z ^ (z >> 30)) * 0xBF58476D1CE4E5B9) & (2 ** 64 - 1)
    z = ((z ^ (z >> 27)) * 0x94D049BB133111EB) & (2 ** 64 - 1)
    z = z ^ (z >> 31)
    assert int(synth.words(0, 0, 0, 1)[0]) == z == 0xE220A8397B1DCDAF


def test_seeds_and_streams_differ():
    a = synth.data(64, seed=0)
    assert a.tobytes() != synth.data(64, seed=1).tobytes()
    assert a.tobytes() != synth.stream_bytes(0, 1, 0, 64).tobytes()


def test_bad_set_and_corruption():
    std = b"ABCDEFGHIJKLMNOPQRSTUVWXYZabcdefghijklmnopqrstuvwxyz0123456789+/"
    bad = synth.bad_set(std)
    assert bad.size == 63 and not (set(bad.tolist()) & (set(std) | {61}))
    pos, b = synth.corruption(16, 1398104, std, seed=0)
    assert len(set(pos.tolist())) == 16 and pos.max() < 1398104
    assert set(b.tolist()) <= set(bad.tolist())


def test_loguniform_lengths():
    L = synth.loguniform_lengths(200000, seed=0)
    assert L.min() >= 1 and L.max() <= 65536
    # mean of a log-uniform on [1, 65537) is (b - a) / ln(b / a) ~ 5909
    assert abs(L.mean() - 65536 / np.log(65537)) / 5909 < 0.03
    assert 0.3 < (L < 48).mean() < 0.4
