#!/bin/bash
# extra bench configs on one GPU (the driver's headline is the default C2 run)
python bench.py --config c4 --steps 2 --warmup 3 > gpurun_out/bench_c4.json 2> gpurun_out/bench_c4.err
python bench.py --config c5 --steps 1 --warmup 3 > gpurun_out/bench_c5.json 2> gpurun_out/bench_c5.err
