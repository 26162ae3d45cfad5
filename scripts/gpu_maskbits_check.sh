set -x
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_maskbits.py -x -q 2>&1 | tail -15 > gpurun_out/mb_tests.log
cat gpurun_out/mb_tests.log
timeout 300 python bench.py > gpurun_out/mb_bench1.json 2>gpurun_out/mb_bench1.err; tail -2 gpurun_out/mb_bench1.err
cat gpurun_out/mb_bench1.json
timeout 300 python bench.py --config C5 > gpurun_out/mb_bench_c5.json 2>&1; tail -1 gpurun_out/mb_bench_c5.json
timeout 1500 python -m pytest tests -x -q -m gpu 2>&1 | tail -5 > gpurun_out/mb_full.log
cat gpurun_out/mb_full.log
