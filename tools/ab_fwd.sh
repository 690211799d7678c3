timeout 1500 python -m pytest tests -m gpu -x -q 2>&1 | tail -3 > gpurun_out/ab_tests.log
python bench.py --no-cpu-baseline > gpurun_out/bench_new.jsonl 2> gpurun_out/bench_new.err
