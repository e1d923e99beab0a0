"""Summarise an ncu report (details page) for the kernels in it."""
import os as _os, sys as _sys  # noqa: E401
_sys.path.insert(0, _os.path.dirname(_os.path.dirname(_os.path.abspath(__file__))))  # ROOT_FOR_TOOLS
import csv, subprocess, sys
KEYS = ['Duration', 'Registers Per Thread', 'Achieved Occupancy', 'Theoretical Occupancy',
        'Block Limit Shared Mem', 'Block Limit Registers', 'Compute (SM) Throughput',
        'DRAM Throughput', 'Dynamic Shared Memory Per Block', 'Grid Size', 'Executed Ipc Active',
        'Achieved Active Warps Per SM']
rep = sys.argv[1]
out = subprocess.run(['ncu', '-i', rep, '--page', 'details', '--csv'], capture_output=True, text=True).stdout
r = list(csv.reader(out.splitlines()))
h = r[0]
cur = None
for row in r[1:]:
    d = dict(zip(h, row))
    if d.get('Metric Name') in KEYS:
        k = (d['ID'], d['Kernel Name'][:40])
        if k != cur:
            print(f"--- {k[0]} {k[1]}")
            cur = k
        print(f"   {d['Metric Name']:32s} {d['Metric Value']} {d['Metric Unit']}")
raw = subprocess.run(['ncu', '-i', rep, '--page', 'raw', '--csv'], capture_output=True, text=True).stdout
r = list(csv.reader(raw.splitlines()))
h = r[0]
for row in r[2:]:
    d = dict(zip(h, row))
    st = {k.replace('smsp__average_warps_issue_stalled_', '').replace('_per_issue_active.ratio', ''): float(v)
          for k, v in d.items() if k.startswith('smsp__average_warps_issue_stalled_') and k.endswith('_per_issue_active.ratio')}
    top = sorted(st.items(), key=lambda x: -x[1])[:6]
    print(d.get('ID'), d.get('Kernel Name', '')[:30], 'stalls/issue:', ', '.join(f"{k}={v:.2f}" for k, v in top),
          '| dram bytes', d.get('dram__bytes_read.sum'), d.get('dram__bytes_write.sum'))
    extra = {k: v for k, v in d.items() if any(t in k for t in ('pipe_fp64', 'smsp__inst_executed.sum', 'bank_conflicts', 'sm__inst_executed_pipe_fp64', 'pipe_shared_cycles', 'l1tex__data_pipe_lsu_wavefronts_mem_shared.sum', 'smsp__thread_inst_executed_per_inst_executed'))}
    for k, v in sorted(extra.items()):
        print(f"      {k} = {v}")
