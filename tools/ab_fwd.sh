for c in 4 3 2; do python bench.py --config $c > gpurun_out/bench_c${c}_v4.jsonl 2> gpurun_out/bench_c${c}_v4.err; done
python bench.py --impl reference > gpurun_out/bench_ref_v3.jsonl 2> gpurun_out/bench_ref_v3.err
python bench.py > gpurun_out/bench_c5_v6.jsonl 2> gpurun_out/bench_c5_v6.err
python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/smoke.log 2>&1
