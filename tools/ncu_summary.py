"""Summarise an ncu --set full report (raw page) for the profiles/ dir."""
import csv
import subprocess
import sys

WANT = ['Kernel Name', 'gpu__time_duration.sum', 'dram__bytes_read.sum', 'dram__bytes_write.sum',
        'dram__throughput.avg.pct_of_peak_sustained_elapsed', 'lts__t_sectors.sum',
        'lts__t_sector_hit_rate.pct', 'l1tex__t_sector_hit_rate.pct',
        'lts__throughput.avg.pct_of_peak_sustained_elapsed', 'sm__warps_active.avg.pct_of_peak_sustained_active',
        'launch__registers_per_thread', 'launch__occupancy_limit_registers', 'launch__grid_size',
        'sm__throughput.avg.pct_of_peak_sustained_elapsed', 'l1tex__throughput.avg.pct_of_peak_sustained_active',
        'smsp__inst_executed.sum', 'l1tex__t_requests_pipe_lsu_mem_global_op_ld.sum',
        'l1tex__t_sectors_pipe_lsu_mem_global_op_ld.sum', 'lts__t_requests_srcunit_tex_op_read.sum',
        'lts__t_sectors_srcunit_tex_op_read.sum', 'smsp__average_warp_latency_issue_stalled_long_scoreboard',
        'smsp__warp_issue_stalled_long_scoreboard_per_warp_active.pct',
        'smsp__warp_issue_stalled_lg_throttle_per_warp_active.pct',
        'smsp__warp_issue_stalled_barrier_per_warp_active.pct',
        'smsp__warp_issue_stalled_membar_per_warp_active.pct',
        'smsp__warp_issue_stalled_no_instruction_per_warp_active.pct',
        'smsp__warp_issue_stalled_wait_per_warp_active.pct',
        'smsp__warp_issue_stalled_short_scoreboard_per_warp_active.pct',
        'smsp__warp_issue_stalled_mio_throttle_per_warp_active.pct',
        'smsp__warp_issue_stalled_math_pipe_throttle_per_warp_active.pct',
        'smsp__issue_active.avg.pct_of_peak_sustained_active',
        'gpc__cycles_elapsed.max', 'sm__cycles_elapsed.avg.per_second']


def summary(rep):
    out = subprocess.run(['ncu', '-i', rep, '--page', 'raw', '--csv'], capture_output=True, text=True).stdout
    rows = list(csv.reader(out.splitlines()))
    hdr, units = rows[0], rows[1]
    idx = {h: i for i, h in enumerate(hdr)}
    res = []
    for r in rows[2:]:
        res.append({w: (r[idx[w]], units[idx[w]]) for w in WANT if w in idx})
    return res


if __name__ == '__main__':
    for d in summary(sys.argv[1]):
        print('----')
        for k, (v, u) in d.items():
            print(f'{k:70s} {v} {u}')


def source_hotspots(rep, kernel_regex, top=25):
    """Per-source-line warp samples / instructions of the first matching kernel."""
    out = subprocess.run(['ncu', '-i', rep, '--page', 'source', '--csv', '--print-source', 'cuda',
                          '-k', f'regex:{kernel_regex}', '--launch-count', '1'],
                         capture_output=True, text=True).stdout
    rows = list(csv.reader(out.splitlines()))
    if not rows:
        return []
    hdr = rows[0]
    res = []
    for r in rows[1:]:
        d = dict(zip(hdr, r))
        try:
            s = float(d.get('Warp Stall Sampling (All Samples)', '0') or 0)
            ins = float(d.get('Instructions Executed', '0') or 0)
        except ValueError:
            continue
        res.append((s, ins, d.get('#', ''), d.get('Source', '')[:110]))
    res.sort(key=lambda x: -x[0])
    return res[:top]
