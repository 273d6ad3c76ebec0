#!/bin/bash
# Multi-GPU final pass (gpurun --gpus 4): strong-scaled C3 / C4 lines at 2 and 4 GPUs, the NCCL
# sharded == single-GPU check at 4, the multi-GPU pytest.
O=gpurun_out/r02mg; mkdir -p $O
for n in 2 4; do
  timeout 900 python bench.py --gpus $n > $O/bench_C3_n$n.json 2> $O/bench_C3_n$n.err
  timeout 1200 python bench.py --gpus $n --config C4 --steps 3 --warmup 2 --no-cpu-baseline > $O/bench_C4_n$n.json 2> $O/bench_C4_n$n.err
done
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29533 tools/multigpu_check.py 4096 3000 > $O/multigpu_check_n4.log 2>&1
timeout 600 python -m pytest tests/test_gpu_multigpu.py -q > $O/pytest_mg.log 2>&1
ls -la $O
