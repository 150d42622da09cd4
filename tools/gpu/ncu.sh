# ncu evidence (run only after the same commands exited 0 without ncu, here with &&)
mkdir -p gpurun_out
T=${TAG:-r02}
python tools/prof_one.py 4 1 > gpurun_out/ncu_plain_$T.log 2>&1 && python tools/prof_one.py 5 1 >> gpurun_out/ncu_plain_$T.log 2>&1 && \
python tools/prof_one.py 3 1 >> gpurun_out/ncu_plain_$T.log 2>&1 && \
python bench.py --steps 2 --warmup 3 --no-t-end --adaptive-horizon 0 --no-cpu-baseline >> gpurun_out/ncu_plain_$T.log 2>&1 && {
ncu --set full --clock-control none --import-source on -k regex:"k_colx|k_rowd|k_dvec|k_colinvw|k_transpose" -s 5 -c 5 -o gpurun_out/ncu_c4_$T python tools/prof_one.py 4 1 > gpurun_out/ncu_log_$T.txt 2>&1
ncu --set full --clock-control none --import-source on -k regex:"k_colx|k_rowd|k_dvec|k_colinvw|k_transpose" -s 5 -c 5 -o gpurun_out/ncu_c5_$T python tools/prof_one.py 5 1 >> gpurun_out/ncu_log_$T.txt 2>&1
ncu --set full --clock-control none --import-source on -k regex:"k_col_fwd|k_row|k_col_inv" -s 3 -c 3 -o gpurun_out/ncu_c3_$T python tools/prof_one.py 3 1 >> gpurun_out/ncu_log_$T.txt 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches_$T.csv python bench.py --steps 2 --warmup 3 --no-t-end --adaptive-horizon 0 --no-cpu-baseline >> gpurun_out/ncu_log_$T.txt 2>&1
}
