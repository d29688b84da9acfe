#!/bin/bash
# Round measurement bundle (run on the GPU box from the repo root): bench lines, launch list, ncu captures.
set -u
OUT=${1:-gpurun_out/round}
mkdir -p $OUT
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,clocks.mem --format=csv > $OUT/gpu.txt 2>&1
python bench.py > $OUT/bench_c5.json 2> $OUT/bench_c5.err
for c in 1 2 3 4; do python bench.py --config $c --steps 3 --warmup 3 --no-cpu-baseline >> $OUT/bench_others.jsonl 2>> $OUT/bench_others.err; done
python bench.py --impl reference --steps 2 --warmup 1 > $OUT/bench_reference.json 2> $OUT/bench_reference.err
python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-guess-run > $OUT/plain_launches.log 2>&1 && \
  ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $OUT/launches.csv \
      python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-guess-run > $OUT/ncu_launches.log 2>&1
python tools/ncu_target.py --config 5 > $OUT/plain_target.log 2>&1 && \
  ncu --set full --clock-control none --import-source on -k regex:"k_newton|k_resjac" -c 2 -o $OUT/prof_c5 \
      python tools/ncu_target.py --config 5 > $OUT/ncu_full.log 2>&1
ls -la $OUT
