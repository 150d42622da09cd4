# per-RHS graph time and per-launch (event-marked) times for the given configs: CFGS="4 5" TAG=x
mkdir -p gpurun_out
python tools/prof_cfg.py ${CFGS:-1 2 3 4 5} > gpurun_out/prof_${TAG:-x}.txt 2>&1
