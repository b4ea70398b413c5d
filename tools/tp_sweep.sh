python tools/sweep_alpha.py --config C2 --grid 2.0:64 > gpurun_out/tp0.log 2>&1
PQRR_TWO_PHASE_W=16 PQRR_R1_DIV=2 python tools/sweep_alpha.py --config C2 --grid 2.0:64 > gpurun_out/tp1.log 2>&1
PQRR_TWO_PHASE_W=16 PQRR_R1_DIV=4 python tools/sweep_alpha.py --config C2 --grid 2.0:64 > gpurun_out/tp2.log 2>&1
PQRR_TWO_PHASE_W=16 PQRR_R1_DIV=8 python tools/sweep_alpha.py --config C2 --grid 2.0:64 > gpurun_out/tp3.log 2>&1
PQRR_R1_DIV=16 python tools/sweep_alpha.py --config C3 --grid 2.0:64 > gpurun_out/tp4.log 2>&1
