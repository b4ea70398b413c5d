cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/r3j_tests.log 2>&1
echo "tests rc=$?" >> gpurun_out/r3j_tests.log
timeout 900 python bench.py --config C2 --no-cpu-baseline --no-recall > gpurun_out/r3j_c2.json 2> gpurun_out/r3j_c2.err
timeout 1200 python bench.py --config C4 --no-cpu-baseline --no-recall > gpurun_out/r3j_c4.json 2> gpurun_out/r3j_c4.err
echo done
