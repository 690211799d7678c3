# ncu --set full (with SASS source) of the steady-state raster forward of phase_times (config 5, 64 views)
CMD="python tools/phase_times.py --config 5 --views 64 --shift 2 --no-count --reps 1 --adaptive --tmask 1"
$CMD > /dev/null 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:"render_fwd_kernel" -s 1 -c 1 -o /tmp/rf $CMD > gpurun_out/rf_ncu.log 2>&1
ncu -i /tmp/rf.ncu-rep --page source --csv --print-source sass > gpurun_out/rf_src.csv 2>/dev/null
ncu -i /tmp/rf.ncu-rep --page raw --csv > gpurun_out/rf_raw.csv 2>/dev/null
