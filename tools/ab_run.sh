#!/bin/bash
# A/B timing of library variants (tools/ab_build.py): ab_run.sh CFG REPS name1 name2 ...
cfg=$1; reps=$2; shift 2
for pass in 1 2; do
  for v in "$@"; do
    if [ "$v" = "main" ]; then lib=paper_2309_09072_b200/lib/liblcsgrid_b200.so; else lib=paper_2309_09072_b200/lib/ab/$v.so; fi
    echo "== $v pass $pass cfg $cfg"
    LCSG_LIB_PATH=$lib python tools/sweep.py $cfg --reps $reps 2>&1 | grep -v "^#"
  done
done
