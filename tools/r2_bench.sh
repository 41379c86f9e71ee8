timeout 900 python bench.py --steps 10 --warmup 3 > gpurun_out/bench2.json 2> gpurun_out/bench2.err
timeout 600 python bench.py --impl reference --steps 5 --warmup 1 > gpurun_out/ref2.json 2> gpurun_out/ref2.err
tail -c 1500 gpurun_out/bench2.err; tail -c 400 gpurun_out/ref2.err
