"""T5: the series-sharded multi-GPU run (one rank per GPU, NCCL all-gather of events) reports
exactly the events of a single-GPU run over all series (same counter-based inputs).

    torchrun --nproc-per-node N --master-addr 127.0.0.1 tools/multigpu_check.py [S] [T]
"""
import os
import sys

import numpy as np
import torch
import torch.distributed as dist

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2410_12588_b200 import bocd, tracegen  # noqa: E402
from paper_2410_12588_b200.distributed import allgather_events, records_to_numpy, shard_range  # noqa: E402


def run(S_lo, S_hi, spec, cfg, T, chunk, dev):
    n = S_hi - S_lo
    b = bocd.BocdBatch(n, R=cfg.R, hazard=cfg.hazard, prior_first_obs=True, prior_cov=cfg.prior_cov,
                       event_mask=3, event_capacity=4096, device=dev.index, series_base=S_lo)
    dt = bocd.DeviceTrace(spec, dev)
    x = torch.empty((n, chunk), dtype=torch.float64, device=dev)
    for t0 in range(0, T, chunk):
        dt.generate(x, S_lo, t0)
        b.update_chunk(x)
    recs, dropped = b.changepoints(device_out=True)
    logR = b.read_posterior()[0]
    b.close()
    assert not dropped
    return recs, logR


def main():
    S = int(sys.argv[1]) if len(sys.argv) > 1 else 4096
    T = int(sys.argv[2]) if len(sys.argv) > 2 else 3000
    rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
    dev = torch.device("cuda", int(os.environ.get("LOCAL_RANK", "0")))
    torch.cuda.set_device(dev)
    dist.init_process_group("nccl", device_id=dev)
    cfg = tracegen.CONFIGS["C3"]
    spec = tracegen.make_spec(cfg, n_series=S)
    lo, hi = shard_range(S, rank, world)
    recs, logR = run(lo, hi, spec, cfg, T, 1000, dev)
    allrec = allgather_events(recs)
    logs = [torch.empty((shard_range(S, r, world)[1] - shard_range(S, r, world)[0], cfg.R), dtype=torch.float64,
                        device=dev) for r in range(world)]
    dist.all_gather(logs, logR)  # posterior check only (not part of the bench data path)
    if rank == 0:
        ref_recs, ref_logR = run(0, S, spec, cfg, T, 1000, dev)
        got, want = records_to_numpy(allrec), records_to_numpy(ref_recs)
        assert np.array_equal(got, want), (len(got), len(want))
        assert torch.equal(torch.cat(logs), ref_logR), "posteriors differ"
        print(f"MULTIGPU OK world={world} S={S} T={T} events={len(got)}", flush=True)
    dist.barrier()
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
