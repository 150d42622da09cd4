mkdir -p gpurun_out
export AGK_LIB=paper_2407_16559_b200/libagk_b200_exp.so
O=gpurun_out/mvar_r02u.txt
for rep in 1 2; do
for v in 0 5 9 10 1; do
  echo "[MVAR=$v] $(AGK_MVAR=$v timeout 300 python tools/prof_size.py 8192 16384 32768 65536 131072 262144 524288 2>&1 | tail -1)" >> $O
done
done
cat $O
