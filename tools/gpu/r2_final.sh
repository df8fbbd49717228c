# round-2 final evidence: tests, bench, ncu launch list (timed region), K1 steady-state ncu --set full
python -c "import __graft_entry__ as g; g.build()" > /dev/null
timeout 1500 python -m pytest tests -m "gpu and not slow" -q > gpurun_out/fin_tests.log 2>&1; echo "tests rc=$?"; tail -1 gpurun_out/fin_tests.log
timeout 600 python bench.py --steps 50 --warmup 5 > gpurun_out/fin_bench.log 2>&1; echo "bench rc=$?"
CMD="python bench.py --steps 5 --warmup 3 --no-e2e --no-cpu-baseline --no-paper-batch"
$CMD > /dev/null 2>&1 && ncu --metrics gpu__time_duration.sum --clock-control none --nvtx --nvtx-include "timed/" --csv $CMD > gpurun_out/fin_launches.csv 2>/dev/null; echo "ncu launches rc=$?"
python tools/ncu_launches.py gpurun_out/fin_launches.csv 5
ncu --set full --clock-control none --import-source on --nvtx --nvtx-include "timed/" -k regex:out_fwd_dw -c 1 -o gpurun_out/fin_k1 $CMD > /dev/null 2>&1; echo "ncu k1 rc=$?"
ncu -i gpurun_out/fin_k1.ncu-rep --page raw --csv 2>/dev/null | python3 -c "
import csv,sys
r=list(csv.reader(sys.stdin)); h=r[0]; d=dict(zip(h,r[2]))
for k in ['gpu__time_duration.sum','dram__bytes_read.sum','dram__bytes_write.sum','dram__throughput.avg.pct_of_peak_sustained_elapsed','sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active','lts__t_sector_hit_rate.pct','launch__registers_per_thread']:
    print(k, d.get(k), r[1][h.index(k)] if k in h else '')
"
rm -f gpurun_out/fin_k1.ncu-rep
