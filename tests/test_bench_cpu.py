"""The bench contract on the CPU (no GPU needed): the reference arm (the oracle on the host
cores) prints exactly one JSON line with the keys the driver reads, for every config; the
oracle sample sizing stays bounded; and the N > 1 launch logic hands the run to
torch.distributed.run only when --gpus > 1 and WORLD_SIZE is unset."""
import json
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import bench  # noqa: E402

KEYS = {"impl", "metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better",
        "scaling", "vs_baseline", "dtype", "data", "config", "cpu_baseline", "e2e", "gpu_launches"}


@pytest.mark.parametrize("config", ["C3", "C2"])
def test_reference_arm_json_line(config):
    p = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--impl", "reference", "--config", config,
                        "--steps", "1", "--warmup", "0", "--ref-steps", "96"],
                       capture_output=True, text=True, timeout=600, cwd=ROOT)
    assert p.returncode == 0, p.stderr[-2000:]
    lines = [ln for ln in p.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1
    d = json.loads(lines[0])
    assert KEYS <= set(d)
    assert d["impl"] == "reference" and d["value"] > 0 and d["higher_is_better"] is True
    assert d["metric"] == bench.METRIC and d["unit"] == bench.UNIT
    assert d["cpu_baseline"]["kind"] == "oracle" and d["cpu_baseline"]["cores"] >= 1
    assert d["e2e"]["h2d_bytes_per_step"] == 0 and d["gpu_launches"] == 0
    assert d["config"]["R"] == {"C3": 1024, "C2": 512}[config]


def test_oracle_sample_is_bounded():
    from paper_2410_12588_b200 import tracegen
    for name, cfg in tracegen.CONFIGS.items():
        n_s, T_s = bench.oracle_sample(cfg)
        assert 1 <= n_s <= cfg.n_series and T_s <= min(cfg.T, 3 * cfg.R)
        # cells of oracle work ~ n_s * T_s * R / 2 stay within ~10-30 s on 16+ cores
        assert n_s * T_s * cfg.R / max(1, bench.host_cores()) < 2.5e9, name


def test_relaunch_only_outside_torchrun(monkeypatch):
    calls = []
    monkeypatch.setattr(bench.subprocess, "call", lambda cmd: calls.append(cmd) or 0)
    monkeypatch.setattr(sys, "argv", ["bench.py", "--gpus", "4", "--steps", "2"])
    monkeypatch.delenv("WORLD_SIZE", raising=False)
    assert bench.main() == 0
    assert calls and calls[0][1:4] == ["-m", "torch.distributed.run", "--nnodes=1"]
    assert "--nproc-per-node=4" in calls[0] and "127.0.0.1" in calls[0]


def test_clock_rules():
    assert bench.clocks_bad({"sm_mhz": 1965, "sm_max_mhz": 1965, "reasons": ["hw_thermal_slowdown"]})
    assert bench.clocks_bad({"sm_mhz": 1200, "sm_max_mhz": 1965, "reasons": []})
    assert not bench.clocks_bad({"sm_mhz": 1900, "sm_max_mhz": 1965, "reasons": ["sw_power_cap"]})
    assert not bench.clocks_bad({"sm_mhz": 1965, "sm_max_mhz": 1965, "reasons": []})
