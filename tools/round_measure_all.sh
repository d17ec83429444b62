bash tools/round_measure.sh > gpurun_out/rm.log 2>&1
for t in memcheck synccheck racecheck; do echo "$t:"; timeout 900 compute-sanitizer --tool $t python tools/sanitize.py 2>&1 | grep -E "ERROR SUMMARY|RACECHECK SUMMARY|Error:|sanitize run" | sort | uniq -c | head -20; done > gpurun_out/sanitizer.txt 2>&1
