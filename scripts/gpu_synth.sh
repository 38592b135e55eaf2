cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_synth.py -q -p no:cacheprovider > gpurun_out/pytest_synth.log 2>&1; echo "synth tests rc=$?"
tail -15 gpurun_out/pytest_synth.log
timeout 600 python scripts/gpu_synth_bench.py > gpurun_out/synth_bench.json 2> gpurun_out/synth_bench.err; echo "synth bench rc=$?"
cat gpurun_out/synth_bench.json; tail -3 gpurun_out/synth_bench.err
timeout 1200 python -m pytest tests -q -m gpu -x -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1; echo "pytest gpu rc=$?"
tail -5 gpurun_out/pytest_gpu.log
