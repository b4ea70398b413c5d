cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "rerank or shortlist or adc or sharded or search or shim" > gpurun_out/r2d_tests.log 2>&1
echo "tests rc=$?" >> gpurun_out/r2d_tests.log
timeout 900 python bench.py --config C2 --no-cpu-baseline --no-recall > gpurun_out/r2d_c2.json 2> gpurun_out/r2d_c2.err
timeout 1200 python bench.py --config C4 --no-cpu-baseline --no-recall > gpurun_out/r2d_c4.json 2> gpurun_out/r2d_c4.err
CMD="python bench.py --config C2 --steps 1 --warmup 1 --no-cpu-baseline --no-recall"
$CMD > gpurun_out/r2d_plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:"rerank_pair" -s 1 -c 1 \
    -o gpurun_out/r2d_prof $CMD > gpurun_out/r2d_ncu.log 2>&1
echo done
