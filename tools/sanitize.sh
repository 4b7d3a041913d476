#!/bin/bash
# compute-sanitizer runs of the round-2 kernels (under gpurun): memcheck of
# the tcgen05 large-batch path and the single-launch route, synccheck of the
# fused C1 decode and the tcgen05 path. Output: gpurun_out/sanitizer/.
O=gpurun_out/sanitizer
mkdir -p $O
CS=compute-sanitizer
REPS=2 timeout 900 $CS --tool memcheck --print-limit 50 python tools/big_probe.py > $O/memcheck_umma_b256.txt 2>&1
B=96 K0=3 REPS=2 timeout 900 $CS --tool memcheck --print-limit 50 python tools/big_probe.py > $O/memcheck_umma_b96.txt 2>&1
timeout 900 $CS --tool memcheck --print-limit 50 python tools/c5_probe.py > $O/memcheck_route_single_launch.txt 2>&1
ITERS=2 timeout 900 $CS --tool synccheck --print-limit 50 python tools/decode_once.py > $O/synccheck_decode_c1.txt 2>&1
REPS=2 timeout 900 $CS --tool synccheck --print-limit 50 python tools/big_probe.py > $O/synccheck_umma_b256.txt 2>&1
echo done
