set -x
CMD="python scripts/dense_one.py fwd 232965 602 16 2"
timeout 300 $CMD > gpurun_out/r2_dr602_plain.txt 2>&1 && \
timeout 600 ncu --set full --clock-control none --import-source on -k regex:dense_rows -c 1 -o gpurun_out/r2_prof_dr602 $CMD > gpurun_out/r2_ncu_dr602.log 2>&1; echo "ncu $?"
cat gpurun_out/r2_dr602_plain.txt
