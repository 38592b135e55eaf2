# launch list + full ncu of the finalize kernels (one GPU)
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
ARGS="--batch 64 --steps 2 --warmup 1 --no-cpu-baseline --no-e2e"
python bench.py $ARGS > gpurun_out/plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv python bench.py $ARGS > gpurun_out/ncu_launch.log 2>&1
echo "launch list rc=$?"
ncu --set full --clock-control none --import-source on -k regex:"k_fuse_ccl|k_output|k_ccl_final|k_pyramid" -c 4 -o gpurun_out/prof_fin -f python bench.py $ARGS > gpurun_out/ncu_full2.log 2>&1
echo "full fin rc=$?"
