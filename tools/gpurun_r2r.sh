cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
CMD="python bench.py --config C4 --steps 1 --warmup 1 --no-cpu-baseline --no-recall"
$CMD > gpurun_out/r2r_plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on \
    -k regex:"rerank_pair|ivf_filter|recheck_smem|lut_pass|select_warp|dtilde_tc|far_bound|topw_certify|assign_tc_kernel|rerank_topk_warp" \
    -s 9 -c 12 -o gpurun_out/r2r_c4 $CMD > gpurun_out/r2r_ncu.log 2>&1
echo "rc=$?" >> gpurun_out/r2r_ncu.log
