# Round profile set (one GPU): bench line, launch list, full ncu of the hot kernels.
cd $GRAFT_REPO_ROOT; OUT=gpurun_out/profile; mkdir -p $OUT
nvidia-smi --query-gpu=name,driver_version,clocks.max.sm,clocks.max.mem --format=csv > $OUT/gpu.txt 2>&1
timeout 900 python -m pytest tests -q -m gpu -p no:cacheprovider > $OUT/pytest_gpu.log 2>&1; echo "pytest rc=$?"
timeout 600 python bench.py > $OUT/bench.json 2> $OUT/bench.err; echo "bench rc=$?"
timeout 600 python bench.py --impl reference --steps 5 --warmup 1 > $OUT/bench_reference.json 2> $OUT/bench_reference.err; echo "ref rc=$?"
ARGS="--batch 64 --steps 2 --warmup 1 --no-cpu-baseline --no-e2e"
python bench.py $ARGS > $OUT/plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $OUT/launches.csv python bench.py $ARGS > $OUT/ncu_launch.log 2>&1
echo "launch list rc=$?"
ncu --set full --clock-control none --import-source on -k regex:k_patches -s 2 -c 1 -o $OUT/k_patches -f python bench.py $ARGS > $OUT/ncu_patches.log 2>&1
echo "full patches rc=$?"
ncu --set full --clock-control none -k regex:"k_fuse_ccl|k_output|k_ccl|k_pyramid" -c 5 -o $OUT/k_other -f python bench.py $ARGS > $OUT/ncu_other.log 2>&1
echo "full other rc=$?"
