cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_cli.py tests/test_gpu_render.py -q -x -p no:cacheprovider > gpurun_out/pytest_cli.log 2>&1; echo "cli tests rc=$?"
tail -30 gpurun_out/pytest_cli.log
