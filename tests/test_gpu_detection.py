"""N3 on the GPU: the detection-ordering property of SPEC.md S:168 (Tables 5-6 of PAPER.md,
P:1121-1159, restated as a property): on a labelled synthetic suite, BOCD + the 10%
verification has a strictly lower false-positive rate than raw BOCD reporting
all suspicious change points (PROB + MAP resets), and raw BOCD's false-negative rate is no
higher than BOCD+V's ("the original BOCD has a lower FNR by reporting all suspicious
change-points but suffers from a high FPR").  Every detector runs through the C ABI
(detection.evaluate).  Suites: the C3 link recipe at CoV 0.05 and 0.1 (measured: raw FPR
0.378 / 0.952 -> BOCD+V 0.0 / 0.089, accuracy 0.785 / 0.459 -> 1.0 / 0.949,
profiles/r02_detection.jsonl)."""
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu
if not torch.cuda.is_available():  # pragma: no cover
    pytest.skip("needs a CUDA device", allow_module_level=True)

from paper_2410_12588_b200 import detection, tracegen  # noqa: E402


@pytest.mark.parametrize("sigma", [0.05, 0.1])
def test_bocd_v_lowers_fpr(sigma):
    cfg = tracegen.CONFIGS["C3"]
    S, T = 512, 6000
    spec = tracegen.make_spec(cfg, n_series=S, T=T, sigma=sigma)
    out = detection.evaluate(spec, cfg, T)
    raw, ver = out["bocd_prob_mapreset"], out["bocd_v_prob_mapreset"]
    assert not out["events_dropped"]
    assert 0 < out["slowed_series"] < S
    assert raw["fp"] > 0
    assert ver["fpr"] < raw["fpr"], (ver, raw)
    assert ver["accuracy"] > raw["accuracy"], (ver, raw)
    assert raw["fnr"] <= ver["fnr"], (ver, raw)
