cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/r2g_tests.log 2>&1
echo "tests rc=$?" >> gpurun_out/r2g_tests.log
timeout 900 python bench.py --config C2 --no-cpu-baseline --no-recall > gpurun_out/r2g_c2.json 2> gpurun_out/r2g_c2.err
timeout 1200 python bench.py --config C4 --no-cpu-baseline --no-recall > gpurun_out/r2g_c4.json 2> gpurun_out/r2g_c4.err
CMD="python bench.py --config C2 --steps 1 --warmup 1 --no-cpu-baseline --no-recall"
$CMD > gpurun_out/r2g_plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:"rerank_pair" -s 1 -c 1 \
    -o gpurun_out/r2g_prof $CMD > gpurun_out/r2g_ncu.log 2>&1
echo done
