#!/bin/bash
# usage: tools/variant_lists.sh CONFIG NAME...  -> gpurun_out/v_CONFIG_NAME.csv
# (NAME = base for the product library, else lib/libpqrr_b200_NAME.so)
CFG=$1; shift
for n in "$@"; do
  if [ "$n" = base ]; then unset PQRR_LIB_PATH; else export PQRR_LIB_PATH=$PWD/paper_1102_3828_b200/lib/libpqrr_b200_$n.so; fi
  timeout 900 ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv \
    --log-file gpurun_out/v_${CFG}_$n.csv python tools/profile_search.py --config $CFG --searches 1 > gpurun_out/v_${CFG}_$n.log 2>&1
  echo "$n rc=$?"
done
