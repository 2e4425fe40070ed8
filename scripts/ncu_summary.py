"""Print the key metrics of an ncu --page details csv (development helper)."""
import csv, sys
keys = ('Duration', 'Compute (SM) Throughput', 'Memory Throughput', 'DRAM Throughput', 'L2 Hit Rate',
        'Issue Slots Busy', 'Warp Cycles Per Issued Instruction', 'Achieved Occupancy', 'Registers Per Thread',
        'Grid Size', 'Block Size', 'Dynamic Shared Memory Per Block', 'L1/TEX Hit Rate')
rows = list(csv.reader(open(sys.argv[1])))
hdr = rows[0]
seen = set()
for r in rows[1:]:
    d = dict(zip(hdr, r))
    k = (d.get('ID'), d.get('Metric Name'))
    if d.get('Metric Name') in keys and k not in seen:
        seen.add(k)
        print(d['ID'], d['Kernel Name'][:50], '|', d['Metric Name'], d['Metric Value'], d['Metric Unit'])
if len(sys.argv) > 2:
    raw = list(csv.reader(open(sys.argv[2])))
    h, u, v = raw[0], raw[1], raw[2]
    for name, unit, val in zip(h, u, v):
        if any(s in name for s in ('dram__bytes_read.sum', 'dram__bytes_write.sum', 'sm__inst_executed_pipe_tensor',
                                   'dmma', 'sm__pipe_fp64', 'smsp__pcsamp_warps_issue_stalled')) and not name.endswith('not_issued'):
            print(name, val, unit)
