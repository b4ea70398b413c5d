cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "rerank or search_matches or adc or group or shim or two_phase" > gpurun_out/r2y_tests.log 2>&1
echo "tests rc=$?" >> gpurun_out/r2y_tests.log
timeout 900 python bench.py --config C2 --no-cpu-baseline --no-recall > gpurun_out/r2y_c2.json 2> gpurun_out/r2y_c2.err
timeout 1200 python bench.py --config C4 --no-cpu-baseline --no-recall > gpurun_out/r2y_c4.json 2> gpurun_out/r2y_c4.err
echo done
