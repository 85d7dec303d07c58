"""On-disk formats against files written by the
reference's own writers (tests/golden/formats, made by make_golden.py
--formats): sample CSV, surrogate spec JSON, `mltune predict` CSV."""

from __future__ import annotations

import json

import numpy as np
import pytest

from conftest import GOLDEN

F = GOLDEN / "formats"


def _tiny():
    import paper_1506_00842_b200 as b
    return b.ParamSpace("tiny", (b.ParamDef("a", (1, 2, 4)), b.ParamDef("b", (0, 1)), b.ParamDef("c", (10, 20, 30, 40))),
                        (b.ValidityRule("max-product", ("a", "c"), bound=80),))


@pytest.mark.parametrize("name", ["samples_convolution.csv", "samples_tiny.csv"])
def test_sample_csv_roundtrip_byte_identical(tmp_path, name):
    from paper_1506_00842_b200.formats import load_samples, measured_indices, save_samples
    space = _tiny() if "tiny" in name else None
    ss = load_samples(F / name, space)
    assert len(ss) > 0
    statuses = {s.outcome.status for s in ss.samples}
    assert "valid" in statuses and statuses - {"valid"}          # both kinds present
    out = tmp_path / name
    save_samples(ss, out)
    assert out.read_bytes() == (F / name).read_bytes()
    assert measured_indices(out, space) == {ss.space.index_of(s.config) for s in ss.samples}


def test_sample_writer_append_and_errors(tmp_path):
    import paper_1506_00842_b200 as b
    from paper_1506_00842_b200.formats import SampleWriter, load_samples
    ss = load_samples(F / "samples_convolution.csv")
    p = tmp_path / "s.csv"
    with SampleWriter(p, ss.space, ss.runner_id) as w:
        for s in ss.samples[:10]:
            w.write(s)
    with SampleWriter(p, ss.space, ss.runner_id, append=True) as w:
        for s in ss.samples[10:]:
            w.write(s)
    assert p.read_bytes() == (F / "samples_convolution.csv").read_bytes()
    bad = tmp_path / "bad.csv"
    lines = (F / "samples_convolution.csv").read_text().splitlines()
    for mutate, line in ((lambda L: ["x"] + L[1:], 1), (lambda L: L[:1] + ["a,b"] + L[2:], 2),
                         (lambda L: L[:2] + [L[2].replace("invalid-launch,", "invalid-launch,0.5")] + L[3:], 3),
                         (lambda L: L[:3] + ["1" + L[3]] + L[4:], 4)):
        bad.write_text("\n".join(mutate(lines)) + "\n")
        with pytest.raises(b.ParseError) as ei:
            load_samples(bad)
        assert f"line {line}" in str(ei.value)
    with pytest.raises(b.ParseError):
        load_samples(F / "samples_tiny.csv")              # not a built-in space: must be passed


def test_surrogate_json_roundtrip():
    from paper_1506_00842_b200.formats import load_surrogate_spec, surrogate_to_json
    p = F / "surrogate_gpu-a_convolution.json"
    spec = load_surrogate_spec(p)
    assert surrogate_to_json(spec) == json.loads(p.read_text())
    assert spec.log_sigma == float(np.sqrt(np.log1p(0.05 ** 2)))


def test_prediction_rows_format_matches_reference():
    from paper_1506_00842_b200.formats import PRED_HEADER, format_prediction_rows
    text = (F / "pred_tiny.csv").read_text()
    assert text.startswith(PRED_HEADER)
    rows = [ln.split(",") for ln in text.splitlines()[1:]]
    idx = np.array([int(r[0]) for r in rows])
    pred = np.array([float(r[1]) for r in rows])
    assert PRED_HEADER + format_prediction_rows(idx, pred) == text
    assert format_prediction_rows([], []) == ""


@pytest.mark.gpu
def test_predictions_csv_from_the_device(gpu_ok, tmp_path):
    """`mltune predict` output from device predictions: same rows, values
    within 1e-13 relative of the reference's numpy file."""
    from paper_1506_00842_b200.formats import write_predictions_csv
    from paper_1506_00842_b200.model import load_model
    for model, ref, idx in (("formats/model_tiny.json", "pred_tiny.csv", None),
                            ("model_conv_k11.json", "pred_conv_4242.csv", [4242])):
        out = tmp_path / ref
        n = write_predictions_csv(load_model(GOLDEN / model), out, indices=idx, chunk=7)
        got = out.read_text().splitlines()
        want = (F / ref).read_text().splitlines()
        assert n == len(want) - 1 and got[0] == want[0]
        for g, w in zip(got[1:], want[1:]):
            gi, gp = g.split(",")
            wi, wp = w.split(",")
            assert gi == wi and float(gp) == pytest.approx(float(wp), rel=1e-13, abs=0)
