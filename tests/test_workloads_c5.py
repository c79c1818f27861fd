"""CPU checks of the C5 generator (workloads/c5.py): its two materialisations (numpy on the host,
torch on a device — here the CPU device) produce the same tokens, segments are the counter
streams of workloads/gen.py, and the shape matches BASELINE configs[4] / SURVEY §8(d)."""
import numpy as np

from workloads.c5 import SEED, c5_large
from workloads.gen import K_PROFILE, K_SYS, run


def test_numpy_and_torch_materialisations_agree():
    warm, timed = c5_large(scale=0.002)
    for seg in (warm, timed):
        s = seg.materialize()
        t, o, u = seg.materialize_torch("cpu", chunk_tokens=1 << 16)
        assert np.array_equal(t.numpy().view(np.uint32)[:s.n_tokens], s.tokens)
        assert np.array_equal(o.numpy().view(np.uint64), s.offsets)
        assert np.array_equal(u.numpy().view(np.uint32), s.users)


def test_segments_are_the_counter_streams():
    warm, timed = c5_large(scale=0.002)
    ws = warm.materialize()
    for j in range(5):
        u = int(ws.users[j])
        p = ws.tokens[int(ws.offsets[j]):int(ws.offsets[j + 1])]
        assert np.array_equal(p[:512], run(SEED, K_SYS, u % 16, 512))
        assert np.array_equal(p[512:768], run(SEED, K_PROFILE, u, 256))


def test_shape_of_the_full_configuration():
    """Full scale without materialising: 4e6 timed requests (50 / 40 / 10 %), ~4.2e9 tokens,
    a warm phase of 200 000 conversations with ~1.08e8 blocks."""
    warm, timed = c5_large(scale=1.0)
    m = timed.meta
    assert timed.n_requests == 4_000_000
    assert (m["continuing"], m["new_sessions"], m["probes"]) == (2_000_000, 1_600_000, 400_000)
    assert 4.0e9 < timed.n_tokens < 4.4e9
    assert warm.n_requests == 200_000 and 1.0e8 < warm.n_blocks() < 1.2e8
