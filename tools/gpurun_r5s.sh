cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
P=${1:-r5s}
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/${P}_tests.log 2>&1; echo "tests rc=$?" >> gpurun_out/${P}_tests.log
timeout 1800 python bench.py > gpurun_out/${P}_c4.json 2> gpurun_out/${P}_c4.err
timeout 1200 python bench.py --config C2 > gpurun_out/${P}_c2.json 2> gpurun_out/${P}_c2.err
echo done
