# C5 sweep bench line (graph path for batches <= 1024) + C4 headline check
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
P=${1:-r5j}
timeout 1500 python bench.py --config C5 > gpurun_out/${P}_c5.json 2> gpurun_out/${P}_c5.err
timeout 1800 python bench.py > gpurun_out/${P}_c4.json 2> gpurun_out/${P}_c4.err
echo done
