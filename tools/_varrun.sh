for v in base t384 fma; do
  DEFORMTRACK_B200_LIB=_variants/$v.so python bench.py --steps 30 --warmup 5 --no-e2e --no-cpu-baseline --no-config5 > gpurun_out/v_$v.json 2> gpurun_out/v_$v.err
done
DEFORMTRACK_B200_LIB=_variants/t384.so python -m pytest tests/test_gpu_solver.py tests/test_gpu_configs.py -x -q > gpurun_out/t384_tests.log 2>&1
DEFORMTRACK_B200_LIB=_variants/fma.so python -m pytest tests/test_gpu_solver.py tests/test_gpu_configs.py tests/test_gpu_coverage.py -q > gpurun_out/fma_tests.log 2>&1
python tools/profile_phases.py --config 2 --frames 6 > gpurun_out/phases_base.txt 2>&1
