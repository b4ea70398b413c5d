cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 600 python tools/sanitize_case.py > gpurun_out/san_synccheck_plain.log 2>&1 && \
timeout 2400 compute-sanitizer --tool synccheck --error-exitcode 9 --print-limit 50 python tools/sanitize_case.py > gpurun_out/san_synccheck.log 2>&1
echo "rc=$?" >> gpurun_out/san_synccheck.log
