# usage: shape_ab.sh "specs" "workloads"   (PSTEREO_TUNE_SPEC values; "-" = planner default)
for v in $1; do for w in $2; do
  if [ "$v" = "-" ]; then S=""; else S="PSTEREO_TUNE_SPEC=$v"; fi
  env $S python scripts/tools/ab_time.py $w | python -c "import sys,json; d=json.loads(sys.stdin.read()); print('$v', d['workload'], round(d['ms_per_step'],4), {k: round(x,4) for k,x in d['stage_ms'].items() if 'patches' in k}, d['digest'])" >> gpurun_out/shape_ab.txt 2>&1
done; done
cat gpurun_out/shape_ab.txt
