cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "rerank or search_matches or group or shim" > gpurun_out/r3c_tests.log 2>&1
echo "tests rc=$?" >> gpurun_out/r3c_tests.log
timeout 1200 python bench.py --config C4 --no-cpu-baseline --no-recall > gpurun_out/r3c_c4.json 2> gpurun_out/r3c_c4.err

echo done
