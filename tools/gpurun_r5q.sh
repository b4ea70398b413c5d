cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 1200 ncu --profile-from-start off --set full --import-source on --clock-control none --cache-control none \
  -k regex:'lut_pass_kernel' -c 1 \
  -o gpurun_out/r5q_lut -f python tools/profile_search.py --config C5 --nq 4096 --searches 1 > gpurun_out/r5q_ncu.log 2>&1
echo done
