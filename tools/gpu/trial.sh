mkdir -p gpurun_out
export AGK_LIB=paper_2407_16559_b200/libagk_b200_exp.so
O=gpurun_out/trial_r02h.txt
for e in "" "AGK_FUSE_STAGES=0" "AGK_PDL=0" "AGK_PDLMASK=127"; do
  echo "== [$e]" >> $O
  env $e python tools/prof_trial.py 5:100 2:50 3:2 --steppers=rkf45,rk4 >> $O 2>&1
done
cat $O
