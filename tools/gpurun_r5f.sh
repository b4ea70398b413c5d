# ncu --set full of the batch-1 hot kernels at C5
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 1200 ncu --profile-from-start off --set full --import-source on --clock-control none --cache-control none \
  -k regex:'lut_pass_kernel|topw_radix|invert_small|sample_threshold|select_topk_kernel|ivf_filter|rerank_topk_kernel' \
  -o gpurun_out/r5f_b1 -f python tools/profile_search.py --config C5 --nq 1 --searches 1 > gpurun_out/r5f_ncu.log 2>&1
echo done
