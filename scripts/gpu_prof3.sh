# full ncu of the finest k_patches (with source) -- one GPU
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
ARGS="--batch 64 --steps 2 --warmup 1 --no-cpu-baseline --no-e2e"
python bench.py $ARGS > gpurun_out/plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:k_patches -s 2 -c 1 -o gpurun_out/prof_patches3 -f python bench.py $ARGS > gpurun_out/ncu_full1.log 2>&1
echo "full patches rc=$?"
