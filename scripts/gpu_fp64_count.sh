# FP64 / conversion instruction counts of the finest k_patches launch (64 config-2 pairs)
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
ARGS="--batch 64 --steps 2 --warmup 1 --no-cpu-baseline --no-e2e"
python bench.py $ARGS > gpurun_out/plain.log 2>&1 || exit 1
M=sm__sass_thread_inst_executed_op_dadd_pred_on.sum,sm__sass_thread_inst_executed_op_dmul_pred_on.sum,sm__sass_thread_inst_executed_op_dfma_pred_on.sum,sm__sass_thread_inst_executed_op_conversion_pred_on.sum,gpu__time_duration.sum
ncu --metrics $M --clock-control none -k regex:k_patches -s 2 -c 1 --csv --log-file gpurun_out/fp64_count.csv python bench.py $ARGS > gpurun_out/ncu_fp64.log 2>&1
echo "fp64 count rc=$?"
cat gpurun_out/fp64_count.csv | tail -6
