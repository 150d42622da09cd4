mkdir -p gpurun_out
for v in 1 0; do AGK_FUSE_STAGES=$v python tools/fuse_check.py > gpurun_out/fuse_check_c$v.txt 2>&1; done
timeout 1500 python -m pytest tests/test_gpu_steps.py tests/test_gpu_run.py tests/test_gpu_parity_runs.py tests/test_gpu_adapter.py -q -p no:cacheprovider > gpurun_out/fuse_tests_c.log 2>&1
