timeout 1800 python -m pytest tests -m gpu -x -q 2>&1 | tail -5 > gpurun_out/ab_tests.log
python bench.py > gpurun_out/bench_c5_v7.jsonl 2> gpurun_out/bench_c5_v7.err
