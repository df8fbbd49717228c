# ncu --set full of the head and bookkeeping kernels (one launch each, inside the timed region)
python -c "import __graft_entry__ as g; g.build()" > /dev/null
CMD="python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu-baseline --no-paper-batch"
$CMD > gpurun_out/ns_plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on --nvtx --nvtx-include "timed/" -k regex:"head_(fwd|bwd|fin)3|commit_ctrl|commit_copy|sample_kernel|adam_kernel|splitk_reduce" -c 8 -o gpurun_out/small_full $CMD > gpurun_out/ncu_small.log 2>&1; echo "ncu rc=$?"
ncu -i gpurun_out/small_full.ncu-rep --page raw --csv 2>/dev/null > gpurun_out/small_raw.csv
ncu -i gpurun_out/small_full.ncu-rep --page source --csv --print-source sass 2>/dev/null > gpurun_out/small_src.csv
python3 - <<'P'
import csv
r=list(csv.reader(open("gpurun_out/small_raw.csv"))); h=r[0]
for row in r[2:]:
    d=dict(zip(h,row))
    def f(c):
        try: return float(d[c].replace(',',''))
        except: return 0.0
    st=sorted([(f(c),c) for c in h if c.startswith('smsp__pcsamp_warps_issue_stalled') and not c.endswith('not_issued')],reverse=True)[:5]
    print(d.get('Kernel Name','')[:28], 'us', f('gpu__time_duration.sum'), 'grid', d.get('launch__grid_size'), 'blk', d.get('launch__block_size'),
          'dram', d.get('dram__bytes_read.sum'), d.get('dram__bytes_write.sum'), 'sm_active%', d.get('sm__cycles_active.avg'), 'cyc', d.get('sm__cycles_elapsed.avg'),
          [(c.replace('smsp__pcsamp_warps_issue_stalled_',''),v) for v,c in st])
P
rm -f gpurun_out/small_full.ncu-rep
