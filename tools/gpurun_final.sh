# Round-end evidence: every bench line on one box, same commit.
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
P=${1:-fin}
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print(\"smoke ok\")" > gpurun_out/${P}_smoke.log 2>&1
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/${P}_tests.log 2>&1; echo "tests rc=$?" >> gpurun_out/${P}_tests.log
timeout 1800 python bench.py > gpurun_out/${P}_c4.json 2> gpurun_out/${P}_c4.err
timeout 1800 python bench.py --impl reference > gpurun_out/${P}_ref_c4.json 2> gpurun_out/${P}_ref_c4.err
timeout 1800 python bench.py --config C2 > gpurun_out/${P}_c2.json 2> gpurun_out/${P}_c2.err
timeout 1800 python bench.py --impl reference --config C2 > gpurun_out/${P}_ref_c2.json 2> gpurun_out/${P}_ref_c2.err
timeout 1200 python bench.py --config C1 > gpurun_out/${P}_c1.json 2> gpurun_out/${P}_c1.err
timeout 1800 python bench.py --config C3 > gpurun_out/${P}_c3.json 2> gpurun_out/${P}_c3.err
timeout 1800 python bench.py --config C5 > gpurun_out/${P}_c5.json 2> gpurun_out/${P}_c5.err
echo done
