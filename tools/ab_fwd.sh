timeout 1800 python -m pytest tests -m gpu -q > gpurun_out/gpu_tests.log 2>&1; tail -3 gpurun_out/gpu_tests.log
python bench.py > gpurun_out/bench_c5_v8.jsonl 2> gpurun_out/bench_c5_v8.err
for c in 4 3 2; do python bench.py --config $c > gpurun_out/bench_c${c}_v6.jsonl 2> gpurun_out/bench_c${c}_v6.err; done
python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/smoke.log 2>&1
