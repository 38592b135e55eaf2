cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_dropin.py tests/test_gpu_metrics.py -q -x -p no:cacheprovider > gpurun_out/quick.log 2>&1; echo "parity rc=$?"; tail -2 gpurun_out/quick.log
timeout 300 python bench.py --steps 20 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/q.json 2>gpurun_out/q.err; echo "bench rc=$? $(python -c "import json;d=json.load(open('gpurun_out/q.json'));print(round(d['value']),d['stage_ms_per_step'])")"
