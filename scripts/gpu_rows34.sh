cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_render.py -q -s -p no:cacheprovider > gpurun_out/pytest_render.log 2>&1; echo "render tests rc=$?"
tail -25 gpurun_out/pytest_render.log
timeout 600 python scripts/gpu_render_bench.py > gpurun_out/render_bench.json 2> gpurun_out/render_bench.err; echo "render bench rc=$?"
cat gpurun_out/render_bench.json; tail -3 gpurun_out/render_bench.err
