#!/bin/bash
# One GPU call's worth of evidence for a round: bench lines (c3 default, momentum, inference, c15b, c2 graph, c3',
# the paper's 3-layer network), the c3' launch list,
# the launch list of the default bench (ncu, cold-cache, serialised) and one ncu --set full capture of the step
# kernel. usage: tools/round_profile.sh <tag>   (writes gpurun_out/<tag>_*)
set -u
tag=${1:-rX}
o=gpurun_out
python bench.py --steps 20 --warmup 5 > $o/${tag}_bench_c3.json 2> $o/${tag}_bench_c3.err
python bench.py --steps 20 --warmup 5 --momentum 0.9 --no-cpu-baseline > $o/${tag}_bench_c3_momentum.json 2>&1
python bench.py --steps 20 --warmup 5 --mode infer > $o/${tag}_bench_c3_infer.json 2>&1
python bench.py --steps 5 --warmup 3 --config c15b --no-cpu-baseline > $o/${tag}_bench_c15b.json 2>&1
python bench.py --steps 200 --warmup 20 --config c2 --graph --no-cpu-baseline > $o/${tag}_bench_c2_graph.json 2>&1
python bench.py --steps 10 --warmup 3 --config c3p > $o/${tag}_bench_c3p.json 2>&1
python bench.py --steps 3 --warmup 3 --config paper3 > $o/${tag}_bench_paper3.json 2>&1
python tools/prof_once.py c3p 1 > $o/${tag}_prof_c3p_plain.log 2>&1 && \
  ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 200 --csv \
      --log-file $o/${tag}_launches_c3p.csv python tools/prof_once.py c3p 1 > $o/${tag}_ncu_c3p.log 2>&1
python bench.py --steps 2 --warmup 3 --no-cpu-baseline > $o/${tag}_plain.log 2>&1 && \
  ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file $o/${tag}_launches_c3.csv \
      python bench.py --steps 2 --warmup 3 --no-cpu-baseline > $o/${tag}_ncu_launches.log 2>&1
python tools/prof_once.py c3 3 > $o/${tag}_prof_plain.log 2>&1 && \
  ncu --set full --clock-control none --import-source on -k regex:step_kernel -s 2 -c 1 -o $o/${tag}_prof \
      python tools/prof_once.py c3 3 > $o/${tag}_ncu_full.log 2>&1
echo done
