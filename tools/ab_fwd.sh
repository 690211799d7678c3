timeout 1800 python -m pytest tests -m gpu -q > gpurun_out/gpu_tests.log 2>&1; tail -3 gpurun_out/gpu_tests.log
python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" 2>&1 | tail -1
python bench.py > gpurun_out/bench_final.jsonl 2> gpurun_out/bench_final.err; tail -c 300 gpurun_out/bench_final.jsonl
