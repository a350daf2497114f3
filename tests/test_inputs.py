"""Pins for the seeded input recipes (inputs/recipe.h), CPU only."""
import numpy as np


def splitmix64_np(z):
    z = z.astype(np.uint64)
    with np.errstate(over="ignore"):
        z = z + np.uint64(0x9E3779B97F4A7C15)
        z = (z ^ (z >> np.uint64(30))) * np.uint64(0xBF58476D1CE4E5B9)
        z = (z ^ (z >> np.uint64(27))) * np.uint64(0x94D049BB133111EB)
    return z ^ (z >> np.uint64(31))


def hashes(seed, start, n):
    i = np.arange(start, start + n, dtype=np.uint64)
    return splitmix64_np((np.uint64(seed) << np.uint64(48)) | i)


def test_int_recipes_match_definition(inputs_mod):
    n = 1 << 16
    h = hashes(0, 123, n)
    want = (((h >> np.uint64(32)) * np.uint64(201)) >> np.uint64(32)).astype(np.int64) - 100
    assert np.array_equal(inputs_mod.fill_host(inputs_mod.I32_U100, 0, 123, n), want)
    h = hashes(2, 0, n)
    assert np.array_equal(inputs_mod.fill_host(inputs_mod.I8_FLAG, 2, 0, n),
                          (h >> np.uint64(63)).astype(np.int8))


def test_u100_and_flag_statistics(inputs_mod):
    n = 1 << 22
    x = inputs_mod.fill_host(inputs_mod.I32_U100, 0, 0, n)
    assert x.min() == -100 and x.max() == 100
    counts = np.bincount(x + 100, minlength=201)
    expect = n / 201
    assert np.all(np.abs(counts - expect) < 6 * np.sqrt(expect))
    f = inputs_mod.fill_host(inputs_mod.I8_FLAG, 2, 0, n)
    assert set(np.unique(f).tolist()) == {0, 1}
    assert abs(int(f.sum()) - n // 2) < 6 * np.sqrt(n / 4)


def test_f16_rne_matches_numpy(inputs_mod):
    """inputs_f32_to_f16 (used by F16_U01) vs numpy's RNE float32->float16 cast,
    on every fp16 value of U[0,1) data and on the ties."""
    n = 1 << 20
    h = hashes(1, 0, n)
    u = (h >> np.uint64(40)).astype(np.float32) * np.float32(2.0 ** -24)
    got = inputs_mod.fill_host(inputs_mod.F16_U01, 1, 0, n)
    assert np.array_equal(got, u.astype(np.float16).view(np.uint16))
    v = got.view(np.float16).astype(np.float64)
    assert v.min() >= 0 and v.max() <= 1.0 and abs(v.mean() - 0.5) < 0.01


def test_normal_recipe_close_to_libm(inputs_mod):
    """Box-Muller with the recipe's own ln/cos agrees with numpy's libm version."""
    n = 1 << 20
    h = hashes(4, 0, n)
    u1 = ((h >> np.uint64(40)) + np.uint64(1)).astype(np.float64) * 2.0 ** -24
    t = ((h >> np.uint64(16)) & np.uint64(0xFFFFFF)).astype(np.float64) * 2.0 ** -24
    ref = np.sqrt(-2.0 * np.log(u1)) * np.cos(2 * np.pi * t)
    got = inputs_mod.fill_host(inputs_mod.F32_NORMAL, 4, 0, n)
    err = np.abs(got.astype(np.float64) - ref)
    assert np.all(err <= 1e-7 * np.maximum(1.0, np.abs(ref)))
    assert np.mean(got == ref.astype(np.float32)) > 0.9999
    assert abs(got.mean()) < 0.01 and abs(got.std() - 1) < 0.01


def test_offsets_and_determinism(inputs_mod):
    for kind in (inputs_mod.I32_U100, inputs_mod.F16_U01, inputs_mod.F32_NORMAL,
                 inputs_mod.I8_FLAG, inputs_mod.I32_FULL):
        a = inputs_mod.fill_host(kind, 7, 0, 300000)
        b = inputs_mod.fill_host(kind, 7, 1000, 5000)
        assert np.array_equal(a[1000:6000], b)
        assert np.array_equal(a, inputs_mod.fill_host(kind, 7, 0, 300000, threads=1))


def test_softmax_rows(inputs_mod):
    P = inputs_mod.fill_host(inputs_mod.F32_SOFTMAX, 3, 0, 6, 131072)
    assert P.shape == (6, 131072)
    assert np.all(P >= 0)
    assert np.all(np.abs(P.astype(np.float64).sum(1) - 1) < 1e-5)
    P2 = inputs_mod.fill_host(inputs_mod.F32_SOFTMAX, 3, 4, 2, 131072)
    assert np.array_equal(P[4:], P2)
    # structure: heavy-tailed rows, max p far above 1/cols
    assert np.all(P.max(1) > 100.0 / 131072)
