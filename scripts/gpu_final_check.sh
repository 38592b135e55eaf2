cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 1200 python -m pytest tests -q -m gpu -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/pytest_gpu.log
grep -i "fail\|error" gpurun_out/pytest_gpu.log | head -5
PSTEREO_BENCH_BACKEND=gloo timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29533 bench.py --gpus 2 --steps 3 --warmup 3 --batch 64 --no-e2e > gpurun_out/bench_n2.json 2> gpurun_out/bench_n2.err; echo "n2 gloo rc=$?"; cat gpurun_out/bench_n2.json | head -c 400; echo
timeout 600 python bench.py --impl reference --gpus 1 --steps 2 --warmup 1 > gpurun_out/ref.json 2>&1; echo "ref rc=$?"; head -c 300 gpurun_out/ref.json; echo
