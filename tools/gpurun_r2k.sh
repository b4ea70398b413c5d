cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
nproc > gpurun_out/r2k_host.txt; df -h /dev/shm /tmp >> gpurun_out/r2k_host.txt; free -g >> gpurun_out/r2k_host.txt
timeout 1500 python bench.py --impl reference > gpurun_out/r2k_ref_c4.json 2> gpurun_out/r2k_ref_c4.err
echo "ref rc=$?" >> gpurun_out/r2k_ref_c4.err
timeout 1500 python bench.py > gpurun_out/r2k_c4.json 2> gpurun_out/r2k_c4.err
echo "ours rc=$?" >> gpurun_out/r2k_c4.err
echo done
