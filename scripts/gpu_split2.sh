cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
for k in 1 2 4; do
  PSTEREO_DEVICE_CHUNKS=$k timeout 300 python bench.py --steps 20 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/split_$k.json 2>gpurun_out/split_$k.err
  echo "chunks=$k rc=$? $(python -c "import json;d=json.load(open('gpurun_out/split_$k.json'));print(round(d['value']),d['ms_per_step'],d['roofline']['frac'],d['stage_ms_per_step'])")"
done
