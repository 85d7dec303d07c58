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
    t, ok = r.run((32, 8, 1, 4, 0, 0, 1, 1, 1), 3)
    assert ok and np.array_equal(r.output(), conv5_box(x))
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
