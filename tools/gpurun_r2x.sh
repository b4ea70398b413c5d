cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 python bench.py --config C2 --no-cpu-baseline --no-recall > gpurun_out/r2x_c2.json 2> gpurun_out/r2x_c2.err
timeout 1200 python bench.py --config C4 --no-cpu-baseline --no-recall > gpurun_out/r2x_c4.json 2> gpurun_out/r2x_c4.err
CMD="python bench.py --config C4 --steps 1 --warmup 1 --no-cpu-baseline --no-recall"
$CMD > gpurun_out/r2x_plain.log 2>&1 && \
ncu --section MemoryWorkloadAnalysis --section SpeedOfLight --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none \
    -k regex:"rerank_pair|recheck_smem|select_warp" -s 3 -c 3 -o gpurun_out/r2x_c4 $CMD > gpurun_out/r2x_ncu.log 2>&1
echo done
