for rep in 1 2; do
SSS_TILE_LISTS_DEV=2 SSS_LIB=variants/libsss_2warp.so python tools/phase_times.py --config 5 --views 64 --shift 2 --no-count --reps 3 --adaptive >> gpurun_out/ab_2w.jsonl 2>&1
python tools/phase_times.py --config 5 --views 64 --shift 2 --no-count --reps 3 --adaptive >> gpurun_out/ab_2w.jsonl 2>&1
done
