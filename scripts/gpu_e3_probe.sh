cd $GRAFT_REPO_ROOT
for spec in "" "e3=256x2x10" "e3=256x2x5" "e3=128x4x5" "e3=128x3x6" "e3=192x2x8" "e3=96x4x6" "e3=64x6x6"; do
  PSTEREO_TUNE_SPEC="$spec" PSTEREO_DEVICE_CHUNKS=1 timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-e2e > /tmp/o.json 2>/dev/null
  echo "spec=[$spec] $(python -c "import json;d=json.load(open('/tmp/o.json'));print(round(d['value']),round(d['stage_ms_per_step']['patches_e3'],4))")"
done
