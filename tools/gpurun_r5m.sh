# ncu --set full of the LUT pass and the filter at C5 batch 16 and batch 1 (graph off so the kernels are plain launches)
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 1200 ncu --profile-from-start off --set full --import-source on --clock-control none --cache-control none \
  -k regex:'lut_pass_kernel|ivf_filter_kernel' \
  -o gpurun_out/r5m_b16 -f python tools/profile_search.py --config C5 --nq 16 --searches 1 > gpurun_out/r5m_ncu.log 2>&1
echo done
