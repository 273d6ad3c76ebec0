#!/bin/bash
# Round-2 multi-GPU pass (run with gpurun --gpus N): strong-scaled C3 and C4 bench lines, the NCCL
# equivalence check (sharded run == one GPU, bit-exact) and the multi-GPU pytest.
N=${N:-2}
O=gpurun_out/r02_mg$N; mkdir -p $O
nvidia-smi --query-gpu=index,name,clocks.sm --format=csv > $O/smi.txt 2>&1
timeout 900 python bench.py --gpus $N --steps 5 --warmup 3 --no-cpu-baseline > $O/bench_C3.json 2> $O/bench_C3.err
timeout 1200 python bench.py --gpus $N --config C4 --steps 3 --warmup 2 --no-cpu-baseline > $O/bench_C4.json 2> $O/bench_C4.err
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 29533 tools/multigpu_check.py 4096 3000 > $O/multigpu_check.log 2>&1
timeout 600 python -m pytest tests/test_gpu_multigpu.py -x -q > $O/pytest_mg.log 2>&1
ls -la $O
