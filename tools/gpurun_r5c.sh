cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
P=${1:-r5d}
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/${P}_tests.log 2>&1; echo "tests rc=$?" >> gpurun_out/${P}_tests.log
timeout 900 python tools/batch_stages.py --config C5 --batches 1,4,16,64,256,1024 > gpurun_out/${P}_stages.log 2>&1
timeout 900 ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --cache-control none --csv --log-file gpurun_out/${P}_c5_b1_launches.csv python tools/profile_search.py --config C5 --nq 1 --searches 1 > gpurun_out/${P}_ncu.log 2>&1
echo done
