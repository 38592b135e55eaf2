cd $GRAFT_REPO_ROOT
for c in 16 32 48 64; do
  PSTEREO_CHUNK_PAIRS=$c timeout 300 python bench.py --steps 20 --warmup 3 --no-cpu-baseline > /tmp/o.json 2>/dev/null
  echo "chunk=$c $(python -c "import json;d=json.load(open('/tmp/o.json'));print(round(d['value']),round(d['e2e']['value']))")"
done
