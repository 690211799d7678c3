timeout 900 python -m pytest tests -m gpu -x -q -k "sghmc or step or graph or variants or loss or relocat or torus or multi" 2>&1 | tail -3 > gpurun_out/ab_tests.log
python bench.py --no-cpu-baseline > gpurun_out/bench_new.jsonl 2> gpurun_out/bench_new.err
