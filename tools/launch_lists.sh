#!/bin/bash
# usage: lst.sh tag  -> launch lists for C2 and C3
ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/l_c3_$1.csv python tools/profile_search.py --config C3 --searches 1 > /dev/null 2>&1
ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/l_c2_$1.csv python tools/profile_search.py --config C2 --searches 1 > /dev/null 2>&1
