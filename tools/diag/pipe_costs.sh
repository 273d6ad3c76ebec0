mkdir -p gpurun_out/pc
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/pc tools/diag/pipe_costs.cu
/tmp/pc > gpurun_out/pc/run.txt
/tmp/pc >> gpurun_out/pc/run.txt
ncu --metrics sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active,l1tex__data_pipe_lsu_wavefronts_mem_shared.sum,smsp__inst_executed.sum,sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active,sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active,sm__cycles_elapsed.avg,smsp__issue_active.avg.pct_of_peak_sustained_active --csv /tmp/pc > gpurun_out/pc/ncu.csv 2>&1
