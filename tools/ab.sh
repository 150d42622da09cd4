#!/bin/bash
# A/B timing of RHS variants: each argument is "ENV=VAL ENV2=VAL2" (use "-" for none)
for spec in "$@"; do
  [ "$spec" = "-" ] && spec=""
  echo "== $spec: $(env $spec python tools/prof_cfg.py ${CFG:-4} 2>&1 | tail -1)"
done
