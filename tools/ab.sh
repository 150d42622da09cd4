#!/bin/bash
# A/B timing of RHS variants: each argument is "ENV=VAL ENV2=VAL2" (use "-" for none).
# The AGK_* knobs are read only by the experiments build: make -C paper_2407_16559_b200 exp
export AGK_LIB=${AGK_LIB:-$(dirname "$0")/../paper_2407_16559_b200/libagk_b200_exp.so}
for spec in "$@"; do
  [ "$spec" = "-" ] && spec=""
  echo "== $spec: $(env $spec python tools/prof_cfg.py ${CFG:-4} 2>&1 | tail -1)"
done
