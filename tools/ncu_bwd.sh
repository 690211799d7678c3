# ncu --set full (with SASS source) of the steady-state raster backward of phase_times (config 5, 64 views)
CMD="python tools/phase_times.py --config 5 --views 64 --shift 2 --no-count --reps 1 --adaptive --tmask 1"
$CMD > /dev/null 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:"render_bwd_kernel" -s 1 -c 1 -o /tmp/rb $CMD > gpurun_out/rb_ncu.log 2>&1
ncu -i /tmp/rb.ncu-rep --page source --csv --print-source sass > gpurun_out/rb_src.csv 2>/dev/null
ncu -i /tmp/rb.ncu-rep --page raw --csv > gpurun_out/rb_raw.csv 2>/dev/null
