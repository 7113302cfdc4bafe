set -x
CMD="python scripts/xent_probe.py 2"
timeout 300 $CMD > gpurun_out/r2_xent_plain.txt 2>&1 && \
timeout 600 ncu --set full --clock-control none --import-source on -k regex:xent -c 2 -o gpurun_out/r2_prof_xent $CMD > gpurun_out/r2_ncu_xent.log 2>&1; echo "ncu $?"
cat gpurun_out/r2_xent_plain.txt
