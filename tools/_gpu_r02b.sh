set -x
python bench.py --gpus 1 --steps 20 --warmup 5 > gpurun_out/r02_bench.json 2> gpurun_out/r02_bench.err
python bench.py --impl reference --gpus 1 --steps 20 --warmup 5 > gpurun_out/r02_bench_reference.json 2> gpurun_out/r02_bench_reference.err
python tools/bench_stereo.py --json gpurun_out/r02_stereo.json > gpurun_out/stereo.log 2>&1
B="python bench.py --steps 3 --warmup 2 --no-e2e --no-cpu-baseline --no-config5"
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r02_launches.csv $B > gpurun_out/ncu_launch.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:"k_observation_normals|k_hamming|k_build_matches|k_preselect_warp|k_preselect_final|k_solve_frame" -s 6 -c 6 -o gpurun_out/r02_frame $B > gpurun_out/ncu_full.log 2>&1
