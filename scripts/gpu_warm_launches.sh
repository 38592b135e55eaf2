# Per-kernel durations with warm caches (ncu --cache-control none), 256-pair bench step
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
ARGS="--batch 256 --steps 1 --warmup 3 --no-cpu-baseline --no-e2e"
PSTEREO_DEVICE_CHUNKS=1 ncu --metrics gpu__time_duration.sum --clock-control none --cache-control none -k regex:"k_(pyramid|patches|fuse|ccl|output)" --csv --log-file gpurun_out/warm.csv python bench.py $ARGS > /dev/null 2>&1
echo rc=$?
python scripts/launches.py gpurun_out/warm.csv
