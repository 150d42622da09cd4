# PDL edge masks at M = 2^20 (experiments build): RHS graph time at configs 4, 5 and config-5 RKF45 trial time
mkdir -p gpurun_out
export AGK_LIB=paper_2407_16559_b200/libagk_b200_exp.so
O=gpurun_out/pdl_${TAG:-x}.txt
for e in "AGK_PDL=0" "AGK_PDLMASK=0" "AGK_PDLMASK=2" "AGK_PDLMASK=8" "AGK_PDLMASK=16" "AGK_PDLMASK=10" "AGK_PDLMASK=18" "AGK_PDLMASK=24" "AGK_PDLMASK=26" "AGK_PDL=0"; do
  echo "[$e] $(env $e python tools/prof_cfg.py 4 2>&1 | cut -c1-30) | $(env $e python tools/prof_trial.py 5:60 2>&1 | tail -1)" >> $O
done
cat $O
