rm -f gpurun_out/ab.jsonl
for rep in 1 2; do for cap in 1536 2048 3072; do echo cap$cap >> gpurun_out/ab.jsonl; python tools/phase_times.py --config 5 --views 64 --shift 2 --no-count --reps 3 --adaptive --tmask 1 --tile-cap $cap >> gpurun_out/ab.jsonl 2>&1; done; done
