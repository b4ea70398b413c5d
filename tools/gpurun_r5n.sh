cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
P=${1:-r5n}
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/${P}_tests.log 2>&1; echo "tests rc=$?" >> gpurun_out/${P}_tests.log
timeout 1500 python bench.py --config C3 > gpurun_out/${P}_c3.json 2> gpurun_out/${P}_c3.err
timeout 1500 python bench.py --config C5 > gpurun_out/${P}_c5.json 2> gpurun_out/${P}_c5.err
echo done
