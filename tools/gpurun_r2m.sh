cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/r2m_tests.log 2>&1
echo "tests rc=$?" >> gpurun_out/r2m_tests.log
timeout 900 python bench.py --config C2 --no-cpu-baseline --no-recall > gpurun_out/r2m_c2.json 2> gpurun_out/r2m_c2.err
timeout 1200 python bench.py --config C4 --no-cpu-baseline --no-recall > gpurun_out/r2m_c4.json 2> gpurun_out/r2m_c4.err
timeout 1500 python tools/sweep_alpha.py --config C4 --grid "1.5:128,1.4:160,1.3:192,1.3:256,1.2:256,1.25:384" > gpurun_out/r2m_sweep.log 2>&1
echo done
