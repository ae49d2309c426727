mkdir -p gpurun_out/r02san; O=gpurun_out/r02san
export LRS_NO_AUTOTUNE=1
timeout 300 python tools/sanitize_run.py > $O/plain.log 2>&1 && \
timeout 1500 compute-sanitizer --tool racecheck --racecheck-report all python tools/sanitize_run.py > $O/racecheck.log 2>&1; echo "racecheck rc=$?" >> $O/rc.txt
tail -5 $O/racecheck.log
