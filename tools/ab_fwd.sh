CMD="python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-next --e2e-steps 1"
K='regex:project_kernel|keys_init4_kernel|radix_hist_kernel|radix_onesweep_kernel|chunk_hist_kernel|column_scan_kernel|bin_scan_kernel|scatter_kernel|tile_mask_kernel|render_fwd_kernel|render_bwd_kernel|project_bwd_kernel|sghmc_kernel'
$CMD > gpurun_out/r02_plain2.log 2>&1 && \
ncu -f --set full --clock-control none --import-source on -k "$K" -s 32 -c 16 -o /tmp/r02_full $CMD > gpurun_out/r02_ncu_full.log 2>&1
ncu -i /tmp/r02_full.ncu-rep --page raw --csv > gpurun_out/r02_full_raw.csv
ncu -i /tmp/r02_full.ncu-rep --page details --csv > gpurun_out/r02_full_details.csv
