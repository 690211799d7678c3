git_lib=paper_2503_10148_b200/build_SSS_BASE1/libsss.so
rm -f gpurun_out/ab.jsonl
for rep in 1 2; do for lib in paper_2503_10148_b200/libsss.so $git_lib; do echo $lib >> gpurun_out/ab.jsonl; SSS_LIB=$lib python bench.py --no-cpu-baseline --no-next --steps 5 >> gpurun_out/ab.jsonl 2>/dev/null; done; done
