#!/bin/bash
# Round-end extra configs on one B200 (under gpurun): the C2 sweep (B x k0
# grid, latency CSV / fit / SVG), the C4 94-layer stack on one GPU, the C5
# router sweep. Output: gpurun_out/$R/.
R=${R:-r02}
O=gpurun_out/$R
mkdir -p $O
timeout 1500 python bench.py --config c2 --out-dir $O/c2 > $O/bench_c2.json 2> $O/bench_c2.err
timeout 900 python bench.py --config c4 --steps 10 --warmup 3 > $O/bench_c4_n1.json 2> $O/bench_c4.err
timeout 600 python bench.py --config c5 > $O/bench_c5.json 2> $O/bench_c5.err
timeout 600 python bench.py --config c3 > $O/bench_c3.json 2> $O/bench_c3.err
echo done
