cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/microbench scripts/microbench.cu && /tmp/microbench > gpurun_out/microbench.txt 2>&1; echo rc=$?
cat gpurun_out/microbench.txt
