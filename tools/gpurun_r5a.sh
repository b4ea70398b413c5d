# small-batch latency analysis at C5 (1B): per-stage times and the batch-1 launch list
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 python tools/batch_stages.py --config C5 --batches 1,4,16,64,256 > gpurun_out/r5a_stages.log 2>&1
timeout 900 ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r5a_c5_b1_launches.csv python tools/profile_search.py --config C5 --nq 1 --searches 1 > gpurun_out/r5a_ncu.log 2>&1
echo done
