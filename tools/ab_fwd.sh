rm -f gpurun_out/ab.jsonl
timeout 900 python -m pytest tests -m gpu -x -q -k "render_bwd or backward or grad or view_groups or tile_list" 2>&1 | tail -3 > gpurun_out/ab_tests.log
timeout 900 env SSS_LIB=paper_2503_10148_b200/build_SSS_BWD_PAIR1/libsss.so python -m pytest tests -m gpu -x -q -k "render_bwd or backward or grad or view_groups or tile_list" 2>&1 | tail -3 >> gpurun_out/ab_tests.log
for rep in 1 2; do for lib in paper_2503_10148_b200/libsss.so paper_2503_10148_b200/build_SSS_*/libsss.so; do echo $lib >> gpurun_out/ab.jsonl; SSS_LIB=$lib python tools/phase_times.py --config 5 --views 64 --shift 2 --no-count --reps 3 --adaptive --tmask 1 >> gpurun_out/ab.jsonl 2>&1; done; done
