"""Summarise an ncu report: key metrics per kernel (reads `ncu -i ... --page details --csv`)."""
import csv
import subprocess
import sys

WANT = ['Duration', 'DRAM Throughput', 'L1/TEX Hit Rate', 'L2 Hit Rate', 'Compute (SM) Throughput',
        'Achieved Occupancy', 'Registers Per Thread', 'Executed Ipc Active', 'Issue Slots Busy', 'No Eligible',
        'Theoretical Occupancy', 'L1/TEX Cache Throughput', 'L2 Cache Throughput',
        'Warp Cycles Per Issued Instruction', 'Avg. Active Threads Per Warp', 'Executed Instructions',
        'Memory Throughput', 'Dynamic Shared Memory Per Block', 'Block Limit Registers']


def main(path):
    out = subprocess.run(['ncu', '-i', path, '--page', 'details', '--csv'], capture_output=True, text=True).stdout
    rows = list(csv.reader(out.splitlines()))
    hdr = rows[0]
    ki, mi, vi, ui = (hdr.index(x) for x in ('Kernel Name', 'Metric Name', 'Metric Value', 'Metric Unit'))
    seen = set()
    for r in rows[1:]:
        if r[mi] in WANT:
            key = (r[ki][:40], r[mi], r[ui])
            if key in seen:
                continue
            seen.add(key)
            print(f"{r[ki][:40]:40s} | {r[mi]:36s} = {r[vi]} {r[ui]}")


if __name__ == '__main__':
    main(sys.argv[1])
