"""N4 on the GPU: falcon_classify_groups against the oracle (oracle/groups.py): medians and
suspicious flags bit-identical, for odd/even group counts up to the 8192 limit."""
import numpy as np
import pytest

from oracle import groups as G

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu
if not torch.cuda.is_available():  # pragma: no cover
    pytest.skip("needs a CUDA device", allow_module_level=True)

from paper_2410_12588_b200 import bocd  # noqa: E402


@pytest.mark.parametrize("B,n", [(1, 1), (3, 2), (5, 4), (64, 7), (128, 64), (32, 1000), (8, 1024), (4, 8192)])
def test_classify_matches_oracle(B, n):
    rng = np.random.default_rng(B * 10007 + n)
    t = rng.lognormal(0.0, 0.1, size=(B, n))
    # a few slow groups per round (20-60% longer transfers) and exact ties
    slow = rng.random((B, n)) < 0.05
    t[slow] *= rng.uniform(1.2, 1.6, size=slow.sum())
    if n >= 4:
        t[:, 1] = t[:, 0]
    flags, med = bocd.classify_groups(torch.from_numpy(t).cuda())
    flags, med = flags.cpu().numpy(), med.cpu().numpy()
    want = G.classify(t)
    for b, (m, f) in enumerate(want):
        assert med[b] == m
        assert flags[b].tolist() == f


def test_spec_examples_and_bad_args():
    t = torch.tensor([[10.0, 10, 10, 12], [10, 10, 11, 11], [7, 7, 7, 7]], dtype=torch.float64, device="cuda")
    flags, med = bocd.classify_groups(t)
    assert med.tolist() == [10.0, 10.5, 7.0]
    assert flags.tolist() == [[False, False, False, True], [False] * 4, [False] * 4]
    with pytest.raises(bocd.N.FalconError):
        bocd.classify_groups(torch.zeros((2, 8193), dtype=torch.float64, device="cuda"))
