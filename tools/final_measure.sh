#!/bin/bash
# GPU call: the full evidence set for DESIGN.md / profiles/ -- GPU tests,
# the default bench line, the reference arm, every config's bench line,
# launch list and one `ncu --set full` summary of its hot kernel.
cd "$(dirname "$0")/.."
O=gpurun_out/final
mkdir -p $O
timeout 1200 python -m pytest tests -m gpu -q > $O/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -1 $O/pytest_gpu.log
python bench.py > $O/bench_default.json 2> $O/bench_default.err; echo "bench rc=$?"
python bench.py --impl reference --steps 2 --warmup 1 > $O/bench_reference.json 2> $O/bench_reference.err; echo "ref rc=$?"
declare -A HOT=([c1]=k_spread_global [c2]=k_interp_bulk [c3]=k_spread_rows3 [c3f]=k_spread_rows3 [c4]=k_spread_rows3 [c5]=k_spread_b2own)
for c in c1 c2 c3 c3f c4 c5; do
  B="python bench.py --config $c --steps 2 --warmup 3 --no-cpu --no-e2e"
  timeout 300 python bench.py --config $c --steps 5 --warmup 3 --no-cpu > $O/bench_$c.json 2> $O/bench_$c.err
  timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches_$c.csv $B > /dev/null 2>&1
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:"${HOT[$c]}" -s 1 -c 1 -o $O/prof_$c $B > $O/ncu_$c.log 2>&1
  python tools/ncu_summary.py $O/prof_$c.ncu-rep > $O/ncu_${c}_summary.txt 2>&1
  python tools/ncu_summary.py $O/prof_$c.ncu-rep "${HOT[$c]}" 2>/dev/null | sed -n '/-- stalls/,$p' >> $O/ncu_${c}_summary.txt
  rm -f $O/prof_$c.ncu-rep
  echo "$c done"
done
