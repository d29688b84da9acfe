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
# every other kernel the five configs launch (ncu --set full, one capture per distinct kernel name)
for c in 1 2 3 4; do
  python tools/ncu_target.py --config $c > $OUT/plain_target_c$c.log 2>&1 && \
    ncu --set full --clock-control none --import-source on -k regex:"k_newton|k_init|k_nb_" -c 4 -o $OUT/prof_c$c -f \
        python tools/ncu_target.py --config $c > $OUT/ncu_full_c$c.log 2>&1
  python tools/ncu_summary.py $OUT/prof_c$c.ncu-rep > $OUT/ncu_full_c$c.md 2>&1 && rm -f $OUT/prof_c$c.ncu-rep
done
# the coarse-grid guess kernels (N1) on c4 shapes, short horizon
python tools/ncu_target.py --config 4 --nt 64 --guess-cf 4 > $OUT/plain_target_guess.log 2>&1 && \
  ncu --set full --clock-control none --import-source on -k regex:"k_spline|k_restrict" -c 8 -o $OUT/prof_guess -f \
      python tools/ncu_target.py --config 4 --nt 64 --guess-cf 4 > $OUT/ncu_full_guess.log 2>&1
python tools/ncu_summary.py $OUT/prof_guess.ncu-rep > $OUT/ncu_full_guess.md 2>&1 && rm -f $OUT/prof_guess.ncu-rep
python tools/ncu_summary.py $OUT/prof_c5.ncu-rep > $OUT/ncu_full_c5.md 2>&1
python tools/ncu_lines.py $OUT/prof_c5.ncu-rep 60 k_newton_ps > $OUT/ncu_lines_k_newton_ps_c5.txt 2>&1
python tools/ncu_summary.py --launches $OUT/launches.csv > $OUT/launches_c5.md 2>&1
ls -la $OUT
