# ncu of the steady-state (truncated) scatter of phase_times --adaptive: launch #3
CMD="python tools/phase_times.py --config 5 --views 64 --shift 2 --no-count --reps 1 --adaptive --tmask 1"
for lib in ${LIBS:-paper_2503_10148_b200/libsss.so}; do
  tag=$(echo $lib | tr '/' '_')
  SSS_LIB=$lib $CMD > /dev/null 2>&1 && \
  SSS_LIB=$lib ncu --set full --clock-control none --import-source on -k regex:"scatter_kernel" -s 3 -c 1 -o /tmp/sc_$tag $CMD > gpurun_out/sc_ncu_$tag.log 2>&1
  ncu -i /tmp/sc_$tag.ncu-rep --page source --csv --print-source sass > gpurun_out/sc_src_$tag.csv 2>/dev/null
  ncu -i /tmp/sc_$tag.ncu-rep --page details --csv > gpurun_out/sc_det_$tag.csv 2>/dev/null
done
