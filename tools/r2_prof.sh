# Evidence refresh: decode-only launch list (default bench) + ncu --set full of K1f and K2w.
set -x
mkdir -p gpurun_out
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"k1_|k2_|k_scan|k_region|k_unpack|k_plan" --csv --log-file gpurun_out/launches_decode.csv python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu --no-cache --no-gather > gpurun_out/launch_bench.log 2>&1
bash tools/ncu_full.sh prof_r02b
ncu -i gpurun_out/prof_r02b.ncu-rep --page source --csv --print-source cuda,sass -k regex:k2_warp > gpurun_out/k2_src.csv 2>/dev/null
ncu -i gpurun_out/prof_r02b.ncu-rep --page source --csv --print-source cuda,sass -k regex:k1_fast > gpurun_out/k1_src.csv 2>/dev/null
ls -la gpurun_out
