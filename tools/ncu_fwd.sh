# ncu --set full (with SASS source) of the bench's raster forward instance (render_fwd_kernel<1,0,1>, config 5)
CMD="python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-next --e2e-steps 1"
$CMD > /dev/null 2>&1 && \
ncu -f --set full --clock-control none --import-source on -k regex:"render_fwd_kernel" -s 3 -c 1 -o /tmp/rf $CMD > gpurun_out/rf_ncu.log 2>&1
ncu -i /tmp/rf.ncu-rep --page source --csv --print-source sass > gpurun_out/rf_src.csv 2>/dev/null
ncu -i /tmp/rf.ncu-rep --page raw --csv > gpurun_out/rf_raw.csv 2>/dev/null
