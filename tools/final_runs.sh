#!/bin/bash
# round-2 final evidence: tests, soak, bench lines, launch lists (run on the GPU box via gpurun)
set -u
O=gpurun_out/final; mkdir -p $O
timeout 1500 python -m pytest tests -m gpu -q > $O/gpu_tests.log 2>&1; tail -1 $O/gpu_tests.log
HC_FUZZ_N=150 HC_FUZZ_SEED=20261019 timeout 1200 python -m pytest tests/test_gpu_fuzz.py -q > $O/fuzz_soak.log 2>&1; tail -1 $O/fuzz_soak.log
timeout 900 python bench.py > $O/bench_default_a.json 2> $O/bench_default_a.err
timeout 900 python bench.py > $O/bench_default_b.json 2> $O/bench_default_b.err
timeout 400 python bench.py --config 2 --steps 50 --warmup 5 > $O/bench_config2.json 2> $O/bench_config2.err
timeout 600 python bench.py --config 4 --steps 10 --warmup 3 --no-cpu-baseline > $O/bench_config4.json 2> $O/bench_config4.err
timeout 900 python bench.py --impl reference --steps 2 --warmup 1 > $O/bench_reference.json 2> $O/bench_reference.err
python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > $O/smoke.log 2>&1; tail -1 $O/smoke.log
for c in 2 3 4; do
  timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 600 --csv --log-file $O/launches_config$c.csv \
    python bench.py --config $c --steps 1 --warmup 3 --no-cpu-baseline --no-config5 > /dev/null 2>&1
done
timeout 900 ncu --set full --import-source on --clock-control none -k regex:k_scan_sk -s 5 -c 1 -o $O/scan_config3 \
  python bench.py --config 3 --steps 1 --warmup 3 --no-cpu-baseline --host-frac 0 --no-config5 > /dev/null 2>&1
echo final-done
