# compute-sanitizer over small cases that launch every kernel family (tools/sanitize_case.py)
mkdir -p gpurun_out/r02san
exec > gpurun_out/r02san/log.txt 2>&1
timeout 300 python tools/sanitize_case.py 2>&1 | tail -4; echo "plain rc=$?"
for tool in memcheck racecheck synccheck initcheck; do
  echo "== $tool"
  timeout 1500 compute-sanitizer --tool $tool --target-processes all --print-limit 20 python tools/sanitize_case.py > gpurun_out/r02san/$tool.txt 2>&1; echo "rc=$?"
  grep -E "ERROR SUMMARY|RACECHECK SUMMARY|case .* ok|sanitize cases ok|Error|hazard" gpurun_out/r02san/$tool.txt | sort | uniq -c | head -30
done
