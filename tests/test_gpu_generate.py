"""The on-device planted generator (rtucker_b200_tensor_generate_device): BASELINE's
N(0,1) planted model + dense Gaussian noise (and config 3's Pareto-scaled factor rows),
generated shard by shard on the GPU (the C5 tensor never exists on one host or GPU)."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def test_noise_free_is_the_reconstruction(oracle, rt):
    shape, ranks = (300, 260, 220), (4, 3, 5)
    t, core, fs = rt.Tensor.generate_device(shape, ranks, 0.0, seed=3, want_model=True)
    x = t.numpy()
    ref = oracle.reconstruct(shape, ranks, core, fs)
    assert np.linalg.norm(x - ref) / np.linalg.norm(ref) < 1e-13
    # N(0,1) model entries
    allv = np.concatenate([core.ravel()] + [f.ravel() for f in fs])
    assert abs(allv.mean()) < 0.1 and abs(allv.std() - 1.0) < 0.1


@pytest.mark.parametrize("P", [2, 3])
def test_shards_equal_the_whole(rt, P):
    shape, ranks = (31, 17, 12), (3, 2, 4)
    whole = rt.Tensor.generate_device(shape, ranks, 0.05, seed=11).numpy()
    parts = [rt.Tensor.generate_device(shape, ranks, 0.05, seed=11, shard=(r, P)).numpy()
             for r in range(P)]
    assert np.array_equal(np.concatenate(parts, axis=0), whole)
    lo, hi = rt.shard_rows(1, P, shape[0])
    assert parts[1].shape == (hi - lo,) + shape[1:]


def test_noise_level(rt):
    shape, ranks, eta = (64, 60, 56), (5, 5, 5), 0.01
    t, core, fs = rt.Tensor.generate_device(shape, ranks, eta, seed=5, want_model=True)
    x0 = rt.Tensor.generate_device(shape, ranks, 0.0, seed=5).numpy()
    noise = t.numpy() - x0
    sigma = eta * np.linalg.norm(x0) / np.sqrt(x0.size)
    assert abs(noise.std() / sigma - 1.0) < 0.01
    assert abs(noise.mean()) < 5 * sigma / np.sqrt(x0.size)


def test_pareto_rows(rt):
    shape, ranks = (400, 300, 8), (4, 4, 2)
    _, _, fs = rt.Tensor.generate_device(shape, ranks, 0.0, seed=7, pareto_alpha=1.5,
                                         want_model=True)
    norms = np.linalg.norm(fs[0], axis=1)
    # heavy-tailed row norms: max / median far above the Gaussian case
    assert norms.max() / np.median(norms) > 10
