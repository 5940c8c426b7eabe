"""Summarise an ncu report: key metrics per kernel + top stall lines."""
import csv
import subprocess
import sys

KEYS = ['gpu__time_duration.sum', 'dram__bytes_read.sum', 'dram__bytes_write.sum',
        'sm__throughput.avg.pct_of_peak_sustained_elapsed',
        'gpu__compute_memory_throughput.avg.pct_of_peak_sustained_elapsed',
        'l1tex__t_sector_hit_rate.pct', 'lts__t_sector_hit_rate.pct',
        'l1tex__t_requests_pipe_lsu_mem_global_op_ld.sum', 'l1tex__t_sectors_pipe_lsu_mem_global_op_ld.sum',
        'l1tex__data_pipe_lsu_wavefronts_mem_shared.sum', 'l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum',
        'sm__inst_executed_pipe_fp64.sum.pct_of_peak_sustained_active',
        'sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active',
        'sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active',
        'smsp__inst_executed.sum', 'sm__warps_active.avg.pct_of_peak_sustained_active',
        'launch__registers_per_thread', 'launch__occupancy_limit_registers', 'launch__occupancy_limit_shared_mem',
        'smsp__issue_active.avg.pct_of_peak_sustained_active', 'lts__t_sectors_op_red.sum', 'lts__t_sectors_op_atom.sum']


def raw(path):
    out = subprocess.run(['ncu', '-i', path, '--page', 'raw', '--csv'], capture_output=True, text=True).stdout
    r = list(csv.reader(out.splitlines()))
    return r[0], r[1], r[2:]


def stalls(path, kernel, top=12):
    out = subprocess.run(['ncu', '-i', path, '--page', 'source', '--csv', '-k', kernel, '--print-source', 'sass'],
                         capture_output=True, text=True).stdout
    rows = list(csv.reader(out.splitlines()))
    hdr = None
    for i, r in enumerate(rows):
        if 'Warp Stall Sampling (All Samples)' in r:
            hdr = i
            break
    if hdr is None:
        return []
    h = rows[hdr]
    si, src = h.index('Warp Stall Sampling (All Samples)'), h.index('Source')
    data = [r for r in rows[hdr + 1:] if len(r) > si and r[si].isdigit()]
    tot = sum(int(r[si]) for r in data) or 1
    data.sort(key=lambda r: -int(r[si]))
    return [(int(r[si]) / tot, r[src].strip()[:70]) for r in data[:top]]


if __name__ == '__main__':
    path = sys.argv[1]
    h, u, rows = raw(path)
    ki = h.index('Kernel Name')
    for row in rows:
        print('==', row[ki][:90])
        for k in KEYS:
            if k in h:
                print(f'   {k:70s} {row[h.index(k)]} {u[h.index(k)]}')
        items = []
        for i, name in enumerate(h):
            if name.startswith('smsp__pcsamp_warps_issue_stalled_') and not name.endswith('not_issued'):
                try:
                    items.append((float(row[i]), name.replace('smsp__pcsamp_warps_issue_stalled_', '')))
                except ValueError:
                    pass
        tot = sum(v for v, _ in items) or 1
        print('   stall reasons:', ', '.join(f'{n} {v / tot:.0%}' for v, n in sorted(items, reverse=True)[:7]))
    if len(sys.argv) > 2:
        for kern in sys.argv[2:]:
            print('-- stalls', kern)
            for frac, s in stalls(path, kern):
                print(f'   {frac:6.1%}  {s}')
