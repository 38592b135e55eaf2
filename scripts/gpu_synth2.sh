cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_synth.py -q -p no:cacheprovider > gpurun_out/pytest_synth.log 2>&1; echo "synth tests rc=$?"; tail -3 gpurun_out/pytest_synth.log
timeout 600 python scripts/gpu_synth_bench.py > gpurun_out/synth_bench.json 2> gpurun_out/synth_bench.err; echo "synth bench rc=$?"; cat gpurun_out/synth_bench.json
ncu --metrics gpu__time_duration.sum --clock-control none -k regex:k_syn -c 8 --csv --log-file gpurun_out/syn_launch.csv python scripts/gpu_synth_bench.py > /dev/null 2>&1; python scripts/launches.py gpurun_out/syn_launch.csv
