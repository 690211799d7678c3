#!/bin/bash
# ncu --set full of the raster kernels (one forward, one backward) of phase_times at config 5, 64 views
CMD="python tools/phase_times.py --config 5 --views 64 --shift 2 --no-count --reps 1 --adaptive"
$CMD > gpurun_out/ras_plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:"render_fwd_kernel|render_bwd_kernel" -s 2 -c 2 -o /tmp/ras $CMD > gpurun_out/ras_ncu.log 2>&1
ncu -i /tmp/ras.ncu-rep --page raw --csv > gpurun_out/ras_raw.csv
ncu -i /tmp/ras.ncu-rep --page source --csv > gpurun_out/ras_src.csv
