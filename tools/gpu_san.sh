# compute-sanitizer, one tool after another over tools/sanitize.py (logs under gpurun_out/)
cd $GRAFT_REPO_ROOT
python tools/sanitize.py > gpurun_out/san_plain.log 2>&1; echo "plain rc=$?" >> gpurun_out/san_plain.log
for tool in memcheck synccheck racecheck initcheck; do
  extra=""
  [ $tool = racecheck ] && extra="--racecheck-report hazard"
  timeout 1500 compute-sanitizer --tool $tool $extra --print-limit 50 python tools/sanitize.py > gpurun_out/san_$tool.log 2>&1
  echo "$tool rc=$?" >> gpurun_out/san_$tool.log
done
