# Round profile set (one GPU): tests, smoke, bench line, reference arm, launch
# list, full ncu of the hot kernels, FP64/XU instruction counts, generator and
# renderer benches. Outputs under gpurun_out/profile.
cd $GRAFT_REPO_ROOT; OUT=gpurun_out/profile; mkdir -p $OUT
nvidia-smi --query-gpu=name,driver_version,clocks.max.sm,clocks.max.mem --format=csv > $OUT/gpu.txt 2>&1
timeout 1200 python -m pytest tests -q -m gpu -p no:cacheprovider > $OUT/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -2 $OUT/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $OUT/smoke.log 2>&1; echo "smoke rc=$?"
timeout 600 python bench.py > $OUT/bench.json 2> $OUT/bench.err; echo "bench rc=$?"
timeout 600 python bench.py --impl reference --steps 5 --warmup 1 > $OUT/bench_reference.json 2> $OUT/bench_reference.err; echo "ref rc=$?"
timeout 600 python scripts/gpu_synth_bench.py > $OUT/synth_bench.json 2>/dev/null; echo "synth bench rc=$?"
timeout 600 python scripts/gpu_render_bench.py > $OUT/render_bench.json 2>/dev/null; echo "render bench rc=$?"
timeout 900 python scripts/gpu_configs_bench.py > $OUT/configs_bench.txt 2>&1; echo "configs bench rc=$?"
ARGS="--batch 64 --steps 2 --warmup 1 --no-cpu-baseline --no-e2e"
python bench.py $ARGS > $OUT/plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $OUT/launches.csv python bench.py $ARGS > $OUT/ncu_launch.log 2>&1
echo "launch list rc=$?"
# unsplit launches for the per-kernel captures (64 pairs per launch)
export PSTEREO_DEVICE_CHUNKS=1
ncu --set full --clock-control none --import-source on -k regex:k_patches -s 2 -c 1 -o $OUT/k_patches -f python bench.py $ARGS > $OUT/ncu_patches.log 2>&1
echo "full patches rc=$?"
M=sm__sass_thread_inst_executed_op_dadd_pred_on.sum,sm__sass_thread_inst_executed_op_dmul_pred_on.sum,sm__sass_thread_inst_executed_op_dfma_pred_on.sum,sm__sass_thread_inst_executed_op_conversion_pred_on.sum,gpu__time_duration.sum
ncu --metrics $M --clock-control none -k regex:k_patches -s 2 -c 1 --csv --log-file $OUT/k_patches_fp64_count.csv python bench.py $ARGS > $OUT/ncu_fp64.log 2>&1
echo "fp64 count rc=$?"
ncu --set full --clock-control none -k regex:"k_fuse_ccl|k_output|k_ccl|k_pyramid" -c 5 -o $OUT/k_other -f python bench.py $ARGS > $OUT/ncu_other.log 2>&1
echo "full other rc=$?"
ncu --set full --clock-control none -k regex:"k_syn|k_render" -c 5 -o $OUT/k_gen -f python scripts/gpu_synth_bench.py > $OUT/ncu_gen.log 2>&1
echo "full gen rc=$?"
