mkdir -p gpurun_out
T=${TAG:-fu1}
timeout 1200 python -m pytest tests/test_gpu_steps.py tests/test_gpu_run.py tests/test_gpu_parity_shapes.py -q -p no:cacheprovider -x > gpurun_out/fuse_tests_$T.log 2>&1
for v in 1 0; do AGK_LIB=paper_2407_16559_b200/libagk_b200_exp.so AGK_FUSE_STAGES=$v timeout 600 python tools/runs.py 2 3 5 --horizon 2:500 3:2 5:20 --steppers rkf45,rk4 --out gpurun_out/fuse_runs_${T}_$v.json > gpurun_out/fuse_runs_${T}_$v.log 2>&1; done
