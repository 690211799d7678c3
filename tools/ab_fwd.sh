timeout 1500 python -m pytest tests -m gpu -x -q 2>&1 | tail -3 > gpurun_out/ab_tests.log
rm -f gpurun_out/ab.jsonl
# the base library needs the base Python binding (48-byte records): A/B through git worktree is not available
# on the box, so only the new build is timed here; compare with the committed numbers
for rep in 1 2; do python tools/phase_times.py --config 5 --views 64 --shift 2 --no-count --reps 3 --adaptive --tmask 1 >> gpurun_out/ab.jsonl 2>&1; done
