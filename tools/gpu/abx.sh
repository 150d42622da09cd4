# A/B of experiment knobs in the experiments build on one box: SPECS="- AGK_PFD=2 ..." CFG="4 5" TAG=x
mkdir -p gpurun_out
export AGK_LIB=paper_2407_16559_b200/libagk_b200_exp.so
O=gpurun_out/abx_${TAG:-x}.txt
for rep in 1 2; do
for spec in ${SPECS:--}; do
  [ "$spec" = "-" ] && e="" || e=$(echo $spec | tr ',' ' ')
  echo "[$spec] $(env $e python tools/variant_hash.py ${CFG:-4 5} 2>&1 | tail -1) | $(env $e python tools/prof_cfg.py ${CFG:-4 5} 2>&1 | tr '\n' ' ')" >> $O
done
done
cat $O
