# full ncu (with source) of one launch of each kernel named in $KERNELS -- one GPU
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
ARGS="--batch 64 --steps 2 --warmup 1 --no-cpu-baseline --no-e2e"
python bench.py $ARGS > gpurun_out/plain.log 2>&1 || { echo "plain bench failed"; exit 1; }
for k in $KERNELS; do
  ncu --set full --clock-control none --import-source on -k regex:$k -s 1 -c 1 -o gpurun_out/prof_$k -f python bench.py $ARGS > gpurun_out/ncu_$k.log 2>&1
  echo "$k rc=$?"
done
