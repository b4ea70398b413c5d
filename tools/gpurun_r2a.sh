cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
nproc > gpurun_out/r2a_nproc.txt; free -g >> gpurun_out/r2a_nproc.txt
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/r2a_tests.log 2>&1
timeout 900 python bench.py > gpurun_out/r2a_c4.json 2> gpurun_out/r2a_c4.err
timeout 900 python bench.py --impl reference > gpurun_out/r2a_ref_c4.json 2> gpurun_out/r2a_ref_c4.err
timeout 900 python bench.py --config C2 > gpurun_out/r2a_c2.json 2> gpurun_out/r2a_c2.err
timeout 900 python bench.py --impl reference --config C2 > gpurun_out/r2a_ref_c2.json 2> gpurun_out/r2a_ref_c2.err
echo done
