# usage: ab.sh "variants" "workloads"
for v in $1; do for w in $2; do
  if [ "$v" = default ]; then L=""; else L="PSTEREO_GPU_LIB=build/var/$v/libpstereo_gpu.so"; fi
  env $L python scripts/tools/ab_time.py $w | python -c "import sys,json; d=json.loads(sys.stdin.read()); print('$v', d['workload'], round(d['ms_per_step'],4), {k: round(x,4) for k,x in d['stage_ms'].items() if 'patches' in k}, d['digest'])" >> gpurun_out/ab.txt 2>&1
done; done
cat gpurun_out/ab.txt
