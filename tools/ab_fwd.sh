for lib in paper_2503_10148_b200/libsss.so variants/libsss_smask20.so variants/libsss_smask18.so variants/libsss_fwd18.so; do echo $lib >> gpurun_out/ab_fwd2.jsonl; SSS_LIB=$lib python tools/phase_times.py --config 5 --views 64 --shift 2 --no-count --reps 3 --adaptive >> gpurun_out/ab_fwd2.jsonl 2>&1; done
python tools/strip_overlap.py 4 >> gpurun_out/ab_fwd2.jsonl 2>&1
