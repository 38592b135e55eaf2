# sweep of k_patches CTA shapes for the round-based schedule (one GPU)
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
for cfg in "0 0 20 2" "0 192 15 2" "0 192 25 2" "0 160 20 2" "0 256 20 2" "0 224 20 2" "0 128 20 3"; do
  set -- $cfg
  if [ "$2" = "0" ]; then unset PSTEREO_TUNE_THREADS; else export PSTEREO_TUNE_THREADS=$2; fi
  PSTEREO_TUNE_PPL10=$3 PSTEREO_TUNE_CTAS=$4 timeout 300 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/tune.log 2>&1
  echo "T=$2 ppl10=$3 ctas=$4: $(python -c "import json; d=json.loads(open('gpurun_out/tune.log').read().splitlines()[-1]); print(round(d['value']), {k: round(v,3) for k,v in d['stage_ms_per_step'].items() if 'patches' in k})")"
done
