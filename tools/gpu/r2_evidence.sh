# final-build evidence: K1 per-tile cycle budget, ncu launch list of the timed region, K1 steady-state ncu --set full
python -c "import __graft_entry__ as g; g.build()" > /dev/null
R=1 bash tools/gpu/tile_ab.sh base
timeout 300 python bench.py --steps 10 --warmup 3 --profile > gpurun_out/ev_prof.log 2>&1; head -c 1500 gpurun_out/ev_prof.log; echo
CMD="python bench.py --steps 5 --warmup 3 --no-e2e --no-cpu-baseline --no-paper-batch"
$CMD > /dev/null 2>&1 && ncu --metrics gpu__time_duration.sum --clock-control none --nvtx --nvtx-include "timed/" --csv $CMD > gpurun_out/ev_launches.csv 2>/dev/null; echo "ncu launches rc=$?"
python tools/ncu_launches.py gpurun_out/ev_launches.csv 5
ncu --set full --clock-control none --import-source on --nvtx --nvtx-include "timed/" -k regex:out_fwd_dw -c 1 -o gpurun_out/ev_k1 $CMD > /dev/null 2>&1; echo "ncu k1 rc=$?"
ncu -i gpurun_out/ev_k1.ncu-rep --page raw --csv 2>/dev/null > gpurun_out/ev_k1_raw.csv
python3 - <<'P'
import csv
r=list(csv.reader(open("gpurun_out/ev_k1_raw.csv"))); h=r[0]; d=dict(zip(h,r[2]))
for k in ['gpu__time_duration.sum','dram__bytes_read.sum','dram__bytes_write.sum','dram__throughput.avg.pct_of_peak_sustained_elapsed','dram__cycles_active.avg.pct_of_peak_sustained_elapsed','sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active','lts__t_sector_hit_rate.pct','launch__registers_per_thread','l1tex__data_pipe_lsu_wavefronts_mem_shared.sum','smsp__inst_executed.sum']:
    print(k, d.get(k), r[1][h.index(k)] if k in h else '')
P
ncu -i gpurun_out/ev_k1.ncu-rep --page details --csv 2>/dev/null > gpurun_out/ev_k1_details.csv
rm -f gpurun_out/ev_k1.ncu-rep
