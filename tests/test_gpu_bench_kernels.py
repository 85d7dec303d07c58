"""The sm_100a benchmark kernels behind the runner protocol: every knob
variant computes the same image as the CPU golden, bit-for-bit; launch
limits come back as invalid-launch; the runner drives autotune."""

from __future__ import annotations

import itertools

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def conv_runner(gpu_ok):
    import paper_1506_00842_b200 as b
    from paper_1506_00842_b200.runners import B200ConvRunner
    rng = np.random.default_rng(5)
    img = rng.random((203, 317), dtype=np.float32)     # odd sizes exercise every border path
    r = B200ConvRunner(b.builtin_space("convolution"), width=317, height=203, image=img, default_repetitions=1)
    yield r, img
    r.close()


@pytest.mark.parametrize("flags", list(itertools.product((0, 1), repeat=5)))
def test_conv_variants_bit_exact(conv_runner, flags):
    from oracle.bench_golden import conv5_box
    r, img = conv_runner
    gold = conv5_box(img)
    for wg, ppt in (((32, 8), (1, 1)), ((16, 4), (2, 4)), ((1, 1), (8, 2)), ((128, 8), (1, 2)), ((4, 64), (4, 1)),
                    ((64, 16), (8, 32)), ((2, 2), (128, 128))):   # CTA blocks larger than the image
        cfg = (wg[0], wg[1], ppt[0], ppt[1]) + tuple(flags)
        t, ok = r.run(cfg, 1)
        tile = (wg[0] * ppt[0] + 4) * (wg[1] * ppt[1] + 4) * 4
        if flags[1] and tile > 227 * 1024:       # use_local tile cannot fit: invalid-launch
            assert not ok
            continue
        assert ok, cfg
        out = r.output()
        assert np.array_equal(out, gold), (cfg, np.abs(out - gold).max())
        assert t > 0


def test_conv_invalid_launches(conv_runner):
    r, _ = conv_runner
    assert r.measure((64, 32, 1, 1, 0, 0, 0, 0, 0)).outcome.status == "invalid-launch"      # 2048 threads
    assert r.measure((128, 128, 1, 1, 0, 0, 0, 0, 0)).outcome.status == "invalid-launch"
    assert r.measure((128, 8, 128, 8, 0, 1, 0, 0, 0)).outcome.status == "invalid-launch"    # tile > 227 KB
    s = r.measure((32, 32, 1, 1, 0, 1, 1, 1, 1))
    assert s.outcome.is_valid and s.outcome.time > 0


def test_conv_4096_input_and_default_image(gpu_ok):
    import paper_1506_00842_b200 as b
    from oracle.bench_golden import conv5_box
    from paper_1506_00842_b200.runners import B200ConvRunner
    r = B200ConvRunner(b.builtin_space("convolution"), width=1024, height=768, seed=3)
    x = r.input()
    assert x.min() >= 0 and x.max() < 1 and x.std() > 0.2
    gold = conv5_box(x)
    # unroll + contiguous rows: the 4-row register-blocked path (and its row tails)
    for cfg in ((32, 8, 1, 4, 0, 0, 1, 1, 1), (32, 4, 1, 4, 0, 1, 1, 0, 1), (32, 8, 1, 8, 0, 0, 0, 0, 1),
                (16, 16, 2, 4, 1, 1, 0, 0, 1), (32, 4, 4, 4, 1, 0, 1, 0, 1), (64, 2, 1, 16, 0, 1, 0, 0, 1),
                (32, 8, 1, 6, 0, 1, 1, 0, 1),
                # use_local + padding on a 16-byte pitch: the TMA-staged tile, incl. tiles taller than one
                # 256-row box and boxes hanging past the padded image
                (32, 32, 1, 16, 0, 1, 1, 1, 1), (8, 64, 4, 8, 0, 1, 1, 0, 0), (252, 1, 1, 100, 0, 1, 1, 0, 1),
                (64, 4, 2, 2, 0, 1, 1, 1, 0),
                # 4 x 4 register blocks with 16-byte shared loads (TMA, manual and texture-staged tiles)
                (16, 8, 4, 4, 0, 1, 1, 0, 1), (16, 8, 8, 4, 0, 1, 0, 0, 1), (8, 8, 4, 8, 1, 1, 0, 0, 1),
                (32, 2, 4, 16, 0, 1, 1, 0, 1)):
        t, ok = r.run(cfg, 3)
        assert ok and np.array_equal(r.output(), gold), cfg
    r.close()


def test_autotune_with_the_b200_runner_on_a_reduced_space(gpu_ok):
    """sample -> measure on the B200 kernel -> device train -> device sweep -> re-measure."""
    import paper_1506_00842_b200 as b
    from paper_1506_00842_b200.runners import B200ConvRunner
    conv = b.builtin_space("convolution")
    sp = b.ParamSpace("conv-reduced", tuple(b.ParamDef(p.name, (1, 8, 64) if len(p.values) == 8 else p.values)
                                             for p in conv.params))
    r = B200ConvRunner(sp, width=512, height=512, default_repetitions=1)
    rep = b.autotune(sp, r, b.TunerConfig(n_train=300, m_candidates=20, k_bag=3, seed=1,
                                          train_cfg=b.TrainConfig(epochs=50, seed=1)))
    assert rep.best_time is not None and rep.best_time > 0
    assert rep.measurements_total == 320
    r.close()


# ---- stereo matching -------------------------------------------------------

@pytest.fixture(scope="module")
def stereo_runner(gpu_ok):
    import paper_1506_00842_b200 as b
    from paper_1506_00842_b200.runners import B200StereoRunner
    rng = np.random.default_rng(11)
    right = rng.integers(0, 256, (61, 97), dtype=np.uint8)
    left = np.roll(right, 6, axis=1)
    left[:, :6] = rng.integers(0, 256, (61, 6), dtype=np.uint8)
    left[20:40, 30:60] = np.roll(right, 3, axis=1)[20:40, 30:60]      # a second disparity region
    r = B200StereoRunner(b.builtin_space("stereo"), width=97, height=61, disparities=16, radius=4,
                         left=left, right=right, default_repetitions=1)
    yield r, left, right
    r.close()


@pytest.mark.parametrize("flags", list(itertools.product((0, 1), repeat=4)))
def test_stereo_variants_bit_exact(stereo_runner, flags):
    from oracle.bench_golden import stereo_sad
    r, left, right = stereo_runner
    gold = stereo_sad(left, right, 16, 4)
    assert (gold == 6).mean() > 0.5 and (gold == 3).any()
    shapes = (((32, 8), (1, 1)), ((16, 4), (2, 4)), ((1, 1), (8, 2)), ((128, 2), (1, 1)), ((8, 16), (4, 8)))
    for ud, ux, uy in itertools.product((1, 2, 4, 8), (1, 2, 4), (1, 2, 4)):
        wg, ppt = shapes[(ud + 3 * ux + 7 * uy) % len(shapes)]    # every unroll combo, rotating CTA shapes
        cfg = (wg[0], wg[1], ppt[0], ppt[1]) + tuple(flags) + (ud, ux, uy)
        t, ok = r.run(cfg, 1)
        assert ok, cfg
        out = r.output()
        assert np.array_equal(out, gold), (cfg, int((out != gold).sum()))
        assert t > 0


def test_stereo_invalid_launches_and_default_pair(gpu_ok):
    import paper_1506_00842_b200 as b
    from oracle.bench_golden import stereo_sad
    from paper_1506_00842_b200.runners import B200StereoRunner
    r = B200StereoRunner(b.builtin_space("stereo"), width=256, height=128, disparities=64, radius=4, seed=2)
    left, right = r.input()
    assert left.std() > 30 and right.std() > 30
    gold = stereo_sad(left, right, 64, 4)
    for cfg in ((16, 16, 1, 1, 0, 0, 1, 1, 4, 2, 2), (32, 4, 2, 2, 1, 1, 0, 0, 8, 4, 1)):
        t, ok = r.run(cfg, 2)
        assert ok and np.array_equal(r.output(), gold)
    # the synthetic pair's disparity field is recovered away from the borders
    assert np.isin(gold[8:-8, 80:-8], (8, 20, 32, 44)).mean() > 0.9
    assert r.measure((64, 32, 1, 1, 0, 0, 0, 0, 1, 1, 1)).outcome.status == "invalid-launch"   # 2048 threads
    # right tile (128*32 + 8 + 63) x (16*16 + 8) bytes > 227 KB
    assert r.measure((128, 16, 32, 16, 0, 0, 0, 1, 1, 1, 1)).outcome.status == "invalid-launch"
    assert r.measure((16, 16, 1, 1, 0, 0, 0, 0, 1, 1, 1)).outcome.is_valid
    with pytest.raises(ValueError):
        r.run((16, 16, 1, 1, 0, 0, 0, 0, 3, 1, 1))
    r.close()


# ---- raycasting ------------------------------------------------------------

@pytest.fixture(scope="module")
def ray_runner(gpu_ok):
    import paper_1506_00842_b200 as b
    from oracle.bench_golden import raycast
    from paper_1506_00842_b200.runners import B200RaycastRunner
    r = B200RaycastRunner(b.builtin_space("raycasting"), width=67, height=53, volume_shape=(48, 40, 56), seed=4,
                          default_repetitions=1)
    gold = raycast(r.volume(), r.transfer(), r.camera(), 67, 53)
    yield r, gold
    r.close()


@pytest.mark.parametrize("flags", list(itertools.product((0, 1), repeat=5)))
def test_raycast_variants_bit_exact(ray_runner, flags):
    r, gold = ray_runner
    assert gold[..., 3].max() > 0.3 and (gold[..., 3] == 0).any()    # a real image with background
    shapes = (((32, 8), (1, 1)), ((16, 4), (2, 4)), ((1, 1), (8, 2)), ((128, 8), (1, 1)), ((4, 64), (4, 1)),
              ((2, 2), (64, 32)))
    for q, unroll in enumerate((1, 2, 4, 8, 16)):
        wg, ppt = shapes[(q + sum(flags)) % len(shapes)]
        cfg = (wg[0], wg[1], ppt[0], ppt[1]) + tuple(flags) + (unroll,)
        t, ok = r.run(cfg, 1)
        if not ok:   # only a 1024-thread CTA may exceed the register file with the deepest unroll
            assert wg[0] * wg[1] == 1024, cfg
            continue
        out = r.output()
        assert np.array_equal(out, gold), (cfg, float(np.abs(out - gold).max()))
        assert t > 0


def test_raycast_host_inputs_and_invalid_launches(gpu_ok):
    import paper_1506_00842_b200 as b
    from oracle.bench_golden import raycast
    from paper_1506_00842_b200.runners import B200RaycastRunner
    rng = np.random.default_rng(3)
    vol = rng.integers(0, 256, (20, 24, 28), dtype=np.uint8)
    tf = rng.random((256, 4), dtype=np.float32) * np.float32(0.3)
    r = B200RaycastRunner(b.builtin_space("raycasting"), width=40, height=30, volume_shape=(28, 24, 20),
                          volume=vol, transfer=tf)
    assert np.array_equal(r.volume(), vol) and np.array_equal(r.transfer(), tf)
    gold = raycast(vol, tf, r.camera(), 40, 30)
    t, ok = r.run((8, 8, 2, 2, 1, 0, 1, 1, 1, 4), 3)
    assert ok and np.array_equal(r.output(), gold)
    assert r.measure((64, 32, 1, 1, 0, 0, 0, 0, 0, 1)).outcome.status == "invalid-launch"
    with pytest.raises(ValueError):
        r.run((8, 8, 1, 1, 0, 0, 0, 0, 0, 3))
    r.close()


def test_raycast_budgeted_screening(gpu_ok):
    """mlt_raybench_set_budget: a configuration far slower than the budget
    stops early and times at about the budget; with the budget off again the
    same configuration renders the full, bit-exact image at its normal time."""
    import paper_1506_00842_b200 as b
    from oracle.bench_golden import raycast
    from paper_1506_00842_b200.runners import B200RaycastRunner
    r = B200RaycastRunner(b.builtin_space("raycasting"), width=512, height=512, volume_shape=(256, 256, 256),
                          seed=2, default_repetitions=1)
    slow = (1, 1, 16, 16, 0, 0, 0, 0, 0, 1)          # one thread per 256 pixels: very slow
    t_full, ok = r.run(slow, 1)
    assert ok and t_full > 4e-3
    r.set_budget(5e-4)
    t_screen, ok = r.run(slow, 1)
    assert ok and 5e-4 <= t_screen < min(0.5 * t_full, 3e-3), (t_screen, t_full)
    r.set_budget(None)
    t_again, ok = r.run(slow, 1)
    assert ok and t_again > 0.8 * t_full
    gold = raycast(r.volume(), r.transfer(), r.camera(), 512, 512)
    assert np.array_equal(r.output(), gold)
    r.close()


def test_stereo_budgeted_screening(gpu_ok):
    """mlt_stereobench_set_budget: as for raycasting -- a slow configuration
    stops early under the budget, and renders the exact disparity map again
    with the budget off."""
    import paper_1506_00842_b200 as b
    from paper_1506_00842_b200.runners import B200StereoRunner
    r = B200StereoRunner(b.builtin_space("stereo"), width=512, height=512, seed=5, default_repetitions=1)
    slow = (1, 1, 16, 16, 0, 0, 0, 0, 1, 1, 1)        # one thread per 256 pixels: very slow
    t_full, ok = r.run(slow, 1)
    assert ok
    ref = r.output().copy()
    r.set_budget(min(2e-4, 0.25 * t_full))
    t_screen, ok = r.run(slow, 1)
    assert ok and t_screen < 0.6 * t_full, (t_screen, t_full)
    r.set_budget(None)
    t_again, ok = r.run(slow, 1)
    assert ok and np.array_equal(r.output(), ref)
    r.close()
