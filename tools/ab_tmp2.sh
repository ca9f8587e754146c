mkdir -p gpurun_out
python tools/mv_probe.py > gpurun_out/mv.log 2>&1 && ncu --set full --clock-control none --import-source on -k regex:nf_matvec -s 1 -c 1 -o gpurun_out/prof_mv2 python tools/mv_probe.py > gpurun_out/ncu_mv.log 2>&1
echo rc=$?
