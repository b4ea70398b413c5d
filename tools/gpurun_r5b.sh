# graph-captured small-batch search: GPU suite + C5 stage/latency lines
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
P=${1:-r5b}
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/${P}_tests.log 2>&1; echo "tests rc=$?" >> gpurun_out/${P}_tests.log
timeout 900 python tools/batch_stages.py --config C5 --batches 1,4,16,64,256,1024 > gpurun_out/${P}_stages.log 2>&1
echo done
