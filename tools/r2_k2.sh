# K2w A/B: parity suite on the new build, then config-3 (+8-layer, config 2) stage times for new and variants/*.so
timeout 1200 python -m pytest tests -m gpu -x -q 2>&1 | tail -4 > gpurun_out/pytest_k2.txt
cat gpurun_out/pytest_k2.txt
bash tools/ab_variants.sh 2>&1 | tee gpurun_out/ab.txt
