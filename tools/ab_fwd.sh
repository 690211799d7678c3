rm -f gpurun_out/ab.jsonl
for rep in 1 2; do for lib in paper_2503_10148_b200/libsss.so paper_2503_10148_b200/build_SSS_*/libsss.so; do echo $lib >> gpurun_out/ab.jsonl; SSS_LIB=$lib python tools/phase_times.py --config 5 --views 64 --shift 2 --no-count --reps 3 --adaptive --tmask 1 >> gpurun_out/ab.jsonl 2>&1; done; done
