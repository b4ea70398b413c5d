cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
for n in base nosample noquant noboth; do
  if [ "$n" = base ]; then unset PQRR_LIB_PATH; else export PQRR_LIB_PATH=$PWD/paper_1102_3828_b200/lib/libpqrr_b200_$n.so; fi
  timeout 900 ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --cache-control none --csv -k regex:lut_pass \
    --log-file gpurun_out/r5y_$n.csv python tools/profile_search.py --config C5 --nq 16 --searches 1 > gpurun_out/r5y_$n.log 2>&1
  echo "$n rc=$?"
done
