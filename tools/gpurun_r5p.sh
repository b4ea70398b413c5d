# launch lists: C5 full batch (65536) and C4, warm caches
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 1500 ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --cache-control none --csv --log-file gpurun_out/r5p_c5_launches.csv python tools/profile_search.py --config C5 --searches 1 > gpurun_out/r5p_c5.log 2>&1
timeout 1500 ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --cache-control none --csv --log-file gpurun_out/r5p_c4_launches.csv python tools/profile_search.py --config C4 --searches 1 > gpurun_out/r5p_c4.log 2>&1
echo done
