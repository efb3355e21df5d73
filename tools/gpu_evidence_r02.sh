# Round-2 final evidence (one GPU): bench lines, launch list, ncu capture of the per-frame
# kernels, configs 1-4 parity + timing, solver phase budget.
set -x
python bench.py --gpus 1 --steps 20 --warmup 5 > gpurun_out/r02_bench.json 2> gpurun_out/r02_bench.err
python bench.py --impl reference --gpus 1 --steps 20 --warmup 5 > gpurun_out/r02_bench_reference.json 2> gpurun_out/r02_bench_reference.err
B="python bench.py --steps 3 --warmup 2 --no-e2e --no-cpu-baseline --no-config5"
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r02_launches.csv $B > gpurun_out/ncu_launch.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:"k_observation_normals|k_hamming|k_preselect_orb|k_solve_frame" -s 4 -c 4 -o gpurun_out/r02_frame $B > gpurun_out/ncu_full.log 2>&1
python tools/run_configs.py --json gpurun_out/r02_configs.json > gpurun_out/configs.log 2>&1
python tools/profile_phases.py --config 2 --frames 8 --json gpurun_out/r02_phases.json > gpurun_out/r02_phases.txt 2>&1
