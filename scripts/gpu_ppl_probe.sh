cd $GRAFT_REPO_ROOT
for spec in "" "e2=128x3x15" "e2=128x3x25" "e2=128x3x30" "e2=128x2x30" "e1=192x2x15" "e1=192x2x25" "e1=192x2x30" "e3=256x2x30"; do
  PSTEREO_TUNE_SPEC="$spec" PSTEREO_DEVICE_CHUNKS=1 timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-e2e > /tmp/o.json 2>/dev/null
  echo "spec=[$spec] $(python -c "import json;d=json.load(open('/tmp/o.json'));s=d['stage_ms_per_step'];print(round(d['value']),round(s['patches_e3'],4),round(s['patches_e2'],4),round(s['patches_e1'],4))")"
done
