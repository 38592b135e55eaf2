# Launch list + full ncu captures of the hot kernels (one GPU).
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
ARGS="--batch 64 --steps 2 --warmup 1 --no-cpu-baseline --no-e2e"
python bench.py $ARGS > gpurun_out/plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv python bench.py $ARGS > gpurun_out/ncu_launch.log 2>&1
echo "launch list rc=$?"
ncu --set full --clock-control none --import-source on -k regex:k_patches -s 2 -c 1 -o gpurun_out/prof_patches -f python bench.py $ARGS > gpurun_out/ncu_full1.log 2>&1
echo "full patches rc=$?"
ncu --set full --clock-control none --import-source on -k regex:"k_ccl|k_fuse|k_output|k_level|k_down|k_gray" -c 9 -o gpurun_out/prof_misc -f python bench.py $ARGS > gpurun_out/ncu_full2.log 2>&1
echo "full misc rc=$?"
python bench.py --steps 10 --warmup 3 > gpurun_out/bench.log 2>&1; echo "bench rc=$?"
tail -1 gpurun_out/bench.log
