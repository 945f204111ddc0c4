mkdir -p gpurun_out
ncu --set full --clock-control none --import-source on -k regex:apply_dmma_kwin -c 1 -o gpurun_out/r50_thin python tools/prof_apply.py 20000 64 2500 > gpurun_out/r50_ncu.log 2>&1
ncu -i gpurun_out/r50_thin.ncu-rep --page raw --csv > gpurun_out/r50_thin_raw.csv 2>&1
ncu -i gpurun_out/r50_thin.ncu-rep --page source --csv > gpurun_out/r50_thin_source.csv 2>&1
rm -f gpurun_out/r50_thin.ncu-rep
tail -2 gpurun_out/r50_ncu.log
