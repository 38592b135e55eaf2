# parity tests + bench + a small sweep of k_patches CTA shapes (one GPU)
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 900 python -m pytest tests -q -m gpu -x -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"
tail -2 gpurun_out/pytest_gpu.log
for cfg in "128 15 2" "128 15 3" "128 25 2" "256 12 1" "96 15 3" "64 20 4" "128 10 3"; do
  set -- $cfg
  PSTEREO_TUNE_THREADS=$1 PSTEREO_TUNE_PPL10=$2 PSTEREO_TUNE_CTAS=$3 timeout 300 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/tune.log 2>&1
  echo "T=$1 ppl10=$2 ctas=$3: $(python -c "import json; d=json.loads(open('gpurun_out/tune.log').read().splitlines()[-1]); print(round(d['value']), {k: round(v,3) for k,v in d['stage_ms_per_step'].items()})")"
done
