#!/bin/bash
# GPU call: per-kernel ncu metrics for every config (time, DRAM bytes and
# GB/s, L2 RED / atomic sectors, L2 / DRAM / FP64 / FMA utilisation, smem
# wavefronts) -> profiles-ready tables + the roofline.traffic refresh, and
# one `ncu --set full` summary per sort kernel of c2.  usage: tools/gpu_evidence.sh [tag]
cd "$(dirname "$0")/.."
T=${1:-r02}
O=gpurun_out/evidence_$T
mkdir -p $O
M=gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sectors_op_red.sum,lts__t_requests_op_red.sum,lts__t_sectors_op_atom.sum,lts__throughput.avg.pct_of_peak_sustained_elapsed,dram__throughput.avg.pct_of_peak_sustained_elapsed,sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active,sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active,l1tex__data_pipe_lsu_wavefronts_mem_shared.sum,smsp__inst_executed.sum
for c in c1 c2 c3 c3f c4 c5; do
  B="python bench.py --config $c --steps 2 --warmup 3 --no-cpu --no-e2e --no-sharded"
  $B > $O/plain_$c.log 2>&1 && \
    timeout 900 ncu --metrics $M --clock-control none --csv --log-file $O/kern_$c.csv $B > $O/ncu_$c.log 2>&1
  python tools/kernel_table.py $O/kern_$c.csv --config $c --update-traffic > $O/kernels_$c.txt 2>&1
  echo "$c rc=$?"
done
cp profiles/traffic.json $O/traffic.json
B="python bench.py --config c2 --steps 2 --warmup 3 --no-cpu --no-e2e --no-sharded"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_setpts|k_scan|k_fill_subprob" -s 7 -c 7 -o $O/prof_sort $B > $O/ncu_sort.log 2>&1
python tools/ncu_summary.py $O/prof_sort.ncu-rep > $O/ncu_c2_sort_summary.txt 2>&1
rm -f $O/prof_sort.ncu-rep
echo evidence done
