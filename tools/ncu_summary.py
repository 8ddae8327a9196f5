"""Export the key per-kernel metrics of an ncu report to CSV (what profiles/ keeps).
usage: python tools/ncu_summary.py report.ncu-rep out.csv"""
import csv
import subprocess
import sys

WANT = ['ID', 'Kernel Name', 'gpu__time_duration.sum', 'dram__bytes_read.sum', 'dram__bytes_write.sum',
        'sm__warps_active.avg.pct_of_peak_sustained_active', 'launch__registers_per_thread',
        'launch__grid_size', 'launch__block_size', 'launch__shared_mem_per_block_dynamic',
        'sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active',
        'sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active',
        'l1tex__t_sector_hit_rate.pct', 'lts__t_sector_hit_rate.pct', 'smsp__inst_executed.sum',
        'l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_ld.sum', 'sm__cycles_elapsed.avg.per_second']


def main(rep, out):
    raw = subprocess.run(['ncu', '-i', rep, '--page', 'raw', '--csv'], capture_output=True,
                         text=True).stdout.splitlines()
    rows = list(csv.reader(raw))
    hdr, units = rows[0], rows[1]
    idx = {h: i for i, h in enumerate(hdr)}
    st = [h for h in hdr if h.startswith('smsp__pcsamp_warps_issue_stalled_') and not h.endswith('not_issued')]
    with open(out, 'w', newline='') as f:
        w = csv.writer(f)
        w.writerow(WANT + ['top_stalls'])
        w.writerow([units[idx[x]] if x in idx else '' for x in WANT] + [''])
        for r in rows[2:]:
            vals = sorted([(float(r[idx[h]] or 0), h.replace('smsp__pcsamp_warps_issue_stalled_', ''))
                           for h in st if r[idx[h]] not in ('', 'n/a')], reverse=True)[:4]
            w.writerow([r[idx[x]] if x in idx else '' for x in WANT] +
                       [';'.join(f"{b}:{int(a)}" for a, b in vals)])


if __name__ == '__main__':
    main(sys.argv[1], sys.argv[2])
