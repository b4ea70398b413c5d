cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 1500 python tools/sweep_alpha.py --config C4 --grid "1.5:128,1.4:160,1.3:192,1.3:256,1.2:256,1.25:384,1.15:384" > gpurun_out/r2l_sweep.log 2>&1
echo done
