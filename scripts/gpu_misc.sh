cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_parity.py -q -x -k "sub_batches or determinism" -p no:cacheprovider > gpurun_out/sub.log 2>&1; echo "sub-batch tests rc=$?"; tail -2 gpurun_out/sub.log
timeout 1500 python scripts/gpu_sweep_bench.py > gpurun_out/sweep.json 2> gpurun_out/sweep.err; echo "sweep rc=$?"; cat gpurun_out/sweep.json; tail -3 gpurun_out/sweep.err
