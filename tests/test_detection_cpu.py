"""Host-side scoring of the detection-accuracy harness (paper_2410_12588_b200/detection.py):
the Table 5-6 definitions on hand-built cases, and the ground truth read from
the generator's episode table."""
import numpy as np

from paper_2410_12588_b200 import detection, tracegen


def test_confusion_table_definitions():
    truth = np.array([1, 1, 1, 0, 0, 0, 0, 0], bool)
    flagged = np.array([1, 1, 0, 1, 0, 0, 0, 0], bool)
    c = detection.confusion(flagged, truth)
    assert (c["tp"], c["fp"], c["tn"], c["fn"]) == (2, 1, 4, 1)
    assert c["accuracy"] == 6 / 8 and c["fpr"] == 1 / 5 and c["fnr"] == 1 / 3
    # a perfect detector and an always-on detector
    assert detection.confusion(truth, truth)["accuracy"] == 1.0
    allon = detection.confusion(np.ones(8, bool), truth)
    assert allon["fpr"] == 1.0 and allon["fnr"] == 0.0


def test_first_flag_and_latency():
    first = detection.first_flag([2, 0, 2, 2], [50, 7, 30, 90], 4)
    assert first.tolist() == [7, -1, 30, -1]
    truth = np.array([True, True, True, False])
    onset = np.array([5, 10, 40, -1])
    lat = detection.latency(first, onset, truth)
    # series 0: 7 - 5 = 2; series 1: never flagged; series 2: flagged before its onset (false alarm)
    assert lat["n"] == 1 and lat["median"] == 2.0


def test_series_truth_from_the_episode_table():
    cfg = tracegen.CONFIGS["C3"]
    spec = tracegen.make_spec(cfg, n_series=64, T=5000)
    slowed, onset = detection.series_truth(spec, 0, 5000)
    for s in range(64):
        eps = [(a, b) for a, b, _ in spec.episodes(s) if min(b, 5000) > max(a, 0)]
        assert slowed[s] == bool(eps)
        if eps:
            assert onset[s] == min(a for a, _ in eps)
        else:
            assert onset[s] == -1
    # the C3 recipe slows about 40% of the links
    assert 0.2 < slowed.mean() < 0.6
