mkdir -p gpurun_out
python -m pytest tests/test_gpu_parity.py tests/test_gpu_real_chase.py -q -x -m gpu > gpurun_out/r45_tests.log 2>&1; tail -2 gpurun_out/r45_tests.log
python bench.py > gpurun_out/r45_bench.json 2> gpurun_out/r45_bench.err; cat gpurun_out/r45_bench.json
