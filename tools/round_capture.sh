#!/bin/bash
# Round-end evidence on one B200 (run under gpurun): GPU tests, the default
# bench line, the reference arm, an ncu launch list of the bench, and one
# ncu --set full capture each of the fused C1 kernel, the tcgen05 FFN and the
# single-launch route. Output: gpurun_out/$R/ (R = round tag, default r02).
R=${R:-r02}
O=gpurun_out/$R
mkdir -p $O
python -m pytest tests -m gpu -q > $O/gpu_tests.txt 2>&1; echo "rc=$?" >> $O/gpu_tests.txt
python bench.py > $O/bench.json 2> $O/bench.err
python bench.py --impl reference --steps 3 --warmup 3 > $O/bench_ref.json 2> $O/bench_ref.err
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches.csv \
  python bench.py --steps 3 --warmup 3 --no-extras --no-cpu-baseline > $O/launches_bench.json 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_ffn_bf16 --launch-skip 2 -c 1 \
  -o $O/prof_fused python tools/decode_once.py > $O/prof_fused.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_ffn_umma --launch-skip 1 -c 1 \
  -o $O/prof_umma python tools/big_probe.py > $O/prof_umma.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_group_route --launch-skip 2 -c 1 \
  -o $O/prof_route python tools/c5_probe.py > $O/prof_route.log 2>&1
echo done
