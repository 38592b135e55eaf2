# parity tests + a sweep of k_patches CTA shapes (one GPU)
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 900 python -m pytest tests -q -m gpu -x -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"
tail -2 gpurun_out/pytest_gpu.log
for cfg in "0 128 15 2" "0 128 15 3" "0 128 15 4" "0 96 15 4" "0 128 10 4" "1 128 15 2" "1 128 15 3" "1 96 15 3" "1 128 10 3" "0 64 20 6"; do
  set -- $cfg
  PSTEREO_TUNE_R64=$1 PSTEREO_TUNE_THREADS=$2 PSTEREO_TUNE_PPL10=$3 PSTEREO_TUNE_CTAS=$4 timeout 300 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/tune.log 2>&1
  echo "R64=$1 T=$2 ppl10=$3 ctas=$4: $(python -c "import json; d=json.loads(open('gpurun_out/tune.log').read().splitlines()[-1]); print(round(d['value']), {k: round(v,3) for k,v in d['stage_ms_per_step'].items()})")"
done
