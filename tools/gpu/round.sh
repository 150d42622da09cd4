# full GPU round: smoke, pytest -m gpu (parity report to gpurun_out/parity_$TAG.jsonl), bench
mkdir -p gpurun_out
export AGK_PARITY_REPORT=gpurun_out/parity_${TAG:-r02a}.jsonl; rm -f $AGK_PARITY_REPORT
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/gpu_${TAG:-r02a}.txt 2>&1
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_${TAG:-r02a}.log 2>&1
timeout 2400 python -m pytest tests -m gpu -q -p no:cacheprovider -rf > gpurun_out/gpu_tests_${TAG:-r02a}.log 2>&1
timeout 900 python bench.py > gpurun_out/bench_${TAG:-r02a}.json 2> gpurun_out/bench_${TAG:-r02a}.err
