mkdir -p gpurun_out/ldsw
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/ldsw tools/diag/lds_wavefronts.cu
/tmp/ldsw
ncu --metrics l1tex__data_pipe_lsu_wavefronts_mem_shared_op_ld.sum,smsp__inst_executed_op_shared_ld.sum,l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_ld.sum --csv /tmp/ldsw > gpurun_out/ldsw/ncu.csv 2>&1
