cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
for B in 1 16; do
timeout 900 ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --cache-control none --csv --log-file gpurun_out/r5x_c5_b${B}_launches.csv python tools/profile_search.py --config C5 --nq $B --searches 1 > gpurun_out/r5x_ncu_$B.log 2>&1
done
echo done
