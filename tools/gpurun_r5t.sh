# ncu --set full of the round-2 streaming selections at C4 (one search)
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 1500 ncu --profile-from-start off --set full --import-source on --clock-control none \
  -k regex:'threshold_warp_kernel|topw_certify_kernel|rerank_topk_warp_kernel|select_warp_kernel' \
  -o gpurun_out/r5t_c4_sel -f python tools/profile_search.py --config C4 --searches 1 > gpurun_out/r5t_ncu.log 2>&1
echo done
