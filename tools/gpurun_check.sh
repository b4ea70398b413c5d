# Quick check of a change on the GPU box: GPU suite, then the bench lines named
# (default: C5 sweep).  usage: gpurun -- 'bash tools/gpurun_check.sh TAG [C4 C2 ...]'
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
P=${1:-chk}; shift
CFGS=${@:-C5}
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/${P}_tests.log 2>&1; echo "tests rc=$?" >> gpurun_out/${P}_tests.log
for c in $CFGS; do
  timeout 1800 python bench.py --config $c > gpurun_out/${P}_$c.json 2> gpurun_out/${P}_$c.err
done
echo done
