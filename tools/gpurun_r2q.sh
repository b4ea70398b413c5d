cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "coarse or search_matches or scale" > gpurun_out/r2q_tests.log 2>&1
echo "tests rc=$?" >> gpurun_out/r2q_tests.log
timeout 1500 python bench.py --config C5 > gpurun_out/r2q_c5.json 2> gpurun_out/r2q_c5.err
echo done
