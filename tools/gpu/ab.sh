# A/B of two built libraries on the same box: A = libagk_b200.so, B = $B (default libagk_b200_ab.so)
mkdir -p gpurun_out
B=${B:-paper_2407_16559_b200/libagk_b200_ab.so}
for i in 1 2 3; do
  echo "A: $(python tools/prof_cfg.py ${CFGS:-4 5} 2>&1 | tr '\n' ' ')" >> gpurun_out/ab_${TAG:-x}.txt
  echo "B: $(AGK_LIB=$B python tools/prof_cfg.py ${CFGS:-4 5} 2>&1 | tr '\n' ' ')" >> gpurun_out/ab_${TAG:-x}.txt
done
