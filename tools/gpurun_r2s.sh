cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
CMD="python bench.py --config C4 --steps 1 --warmup 1 --no-cpu-baseline --no-recall"
$CMD > gpurun_out/r2s_plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on \
    -k regex:"rerank_pair|ivf_filter|recheck_smem|lut_pass|select_warp|dtilde_tc|far_bound|topw_certify|rerank_topk_warp" \
    -s 11 -c 11 -o gpurun_out/r2s_c4 $CMD > gpurun_out/r2s_ncu.log 2>&1
echo "rc=$?" >> gpurun_out/r2s_ncu.log
CMD2="python bench.py --config C2 --steps 1 --warmup 1 --no-cpu-baseline --no-recall"
$CMD2 > gpurun_out/r2s_plain2.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r2s_c2_launches.csv $CMD2 > gpurun_out/r2s_ncu2.log 2>&1
echo "rc2=$?" >> gpurun_out/r2s_ncu.log
