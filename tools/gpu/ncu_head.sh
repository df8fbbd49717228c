# ncu --set full of the fused head kernels (one launch each, inside the timed region)
CMD="python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu-baseline --no-paper-batch"
$CMD > gpurun_out/nh_plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on --nvtx --nvtx-include "timed/" -k regex:"head_(fwd|bwd|fin)3" -c 3 -o gpurun_out/head_full $CMD > gpurun_out/ncu_head.log 2>&1; echo "ncu rc=$?"
ncu -i gpurun_out/head_full.ncu-rep --page details --csv 2>/dev/null | grep -E '"(Duration|Registers Per Thread|Achieved Occupancy|Memory Throughput|Compute \(SM\) Throughput|L2 Hit Rate|Warp Cycles Per Issued Instruction)"' | cut -d, -f5,13-16
ncu -i gpurun_out/head_full.ncu-rep --page raw --csv 2>/dev/null | python3 -c "
import csv,sys
r=list(csv.reader(sys.stdin))
h=r[0]
want=[c for c in h if c.startswith('smsp__average_warp_latency_issue_stalled') or c.startswith('smsp__pcsamp_warps_issue_stalled')]
for row in r[2:]:
    d=dict(zip(h,row))
    st=sorted([(float(d[c].replace(',','')) if d[c] not in ('','n/a') else 0,c) for c in h if c.startswith('smsp__pcsamp_warps_issue_stalled') and not c.endswith('not_issued')],reverse=True)[:6]
    print(d.get('Kernel Name','')[:30], d.get('gpu__time_duration.sum'), [(c.replace('smsp__pcsamp_warps_issue_stalled_',''),v) for v,c in st])
"
