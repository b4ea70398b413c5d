cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "bound or two_phase or search_matches or coarse" > gpurun_out/r2u_tests.log 2>&1
echo "tests rc=$?" >> gpurun_out/r2u_tests.log
timeout 1200 python bench.py --config C4 --no-cpu-baseline --no-recall > gpurun_out/r2u_c4.json 2> gpurun_out/r2u_c4.err
timeout 1500 python bench.py --config C5 > gpurun_out/r2u_c5.json 2> gpurun_out/r2u_c5.err
echo done
