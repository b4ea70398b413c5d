cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
CMD="python bench.py --config C2 --steps 1 --warmup 1 --no-cpu-baseline --no-recall"
$CMD > gpurun_out/r2c_plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:"rerank_pair|recheck_smem|ivf_filter" -s 3 -c 3 \
    -o gpurun_out/r2c_prof $CMD > gpurun_out/r2c_ncu.log 2>&1
echo "rc=$?"
