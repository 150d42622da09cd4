# full-horizon device runs (time to t_end) with the reference's per-RHS CPU time for extrapolation:
#   PART=a: configs 1, 2 (three schemes) and config 3; PART=b: config 5 with the three schemes
mkdir -p gpurun_out
T=${TAG:-r02}
if [ "${PART:-a}" = "a" ]; then
python tools/runs.py 1 2 --steppers rk2,rk4,rkf45 --cpu --out gpurun_out/runs_${T}_c12.json > gpurun_out/runs_${T}_c12.log 2>&1
python tools/runs.py 3 --steppers rkf45 --cpu --out gpurun_out/runs_${T}_c3.json > gpurun_out/runs_${T}_c3.log 2>&1
else
python tools/runs.py 5 --steppers rkf45,rk2,rk4 --cpu --out gpurun_out/runs_${T}_c5.json > gpurun_out/runs_${T}_c5.log 2>&1
fi
