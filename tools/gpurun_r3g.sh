cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 600 python tools/profile_search.py --config C4 --searches 1 > gpurun_out/r3g_plain.log 2>&1
echo "plain rc=$?" >> gpurun_out/r3g_plain.log
timeout 1500 ncu --set full --clock-control none --import-source on --profile-from-start off \
  -k regex:"recheck_lut|ivf_filter" -c 2 -o gpurun_out/r3g_c4 -f \
  python tools/profile_search.py --config C4 --searches 1 > gpurun_out/r3g_ncu.log 2>&1
echo "ncu rc=$?" >> gpurun_out/r3g_ncu.log
