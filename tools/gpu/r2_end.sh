# end-of-round evidence on the final build: GPU tests, bench, launch list, K1 ncu --set full, tile budget
python -c "import __graft_entry__ as g; g.build()" > /dev/null
timeout 1500 python -m pytest tests -m "gpu and not slow" -q > gpurun_out/e_tests.log 2>&1; echo "tests rc=$?"; tail -2 gpurun_out/e_tests.log
timeout 300 python bench.py > gpurun_out/e_bench.log 2>&1; echo "bench rc=$?"
python3 -c "
import json; l=[x for x in open('gpurun_out/e_bench.log') if x.startswith('{')][-1]; d=json.loads(l)
print(round(d['value']), d['ms_per_step'], d['gpu_launches'], round(d['roofline']['frac'],3), round(d['e2e']['value']), round(d['paper_batch_b10']['samples_per_s']), d['clocks'], d['windows_samples_per_s'])"
R=1 bash tools/gpu/tile_ab.sh base
CMD="python bench.py --steps 5 --warmup 3 --no-e2e --no-cpu-baseline --no-paper-batch"
$CMD > /dev/null 2>&1 && ncu --metrics gpu__time_duration.sum --clock-control none --nvtx --nvtx-include "timed/" --csv $CMD > gpurun_out/e_launches.csv 2>/dev/null; echo "ncu launches rc=$?"
python tools/ncu_launches.py gpurun_out/e_launches.csv 5
ncu --set full --clock-control none --import-source on --nvtx --nvtx-include "timed/" -k regex:out_fwd_dw -c 1 -o gpurun_out/e_k1 $CMD > /dev/null 2>&1; echo "ncu k1 rc=$?"
ncu -i gpurun_out/e_k1.ncu-rep --page raw --csv 2>/dev/null > gpurun_out/e_k1_raw.csv
python3 - <<'P'
import csv
r=list(csv.reader(open("gpurun_out/e_k1_raw.csv"))); h=r[0]; d=dict(zip(h,r[2]))
for k in ['gpu__time_duration.sum','dram__bytes_read.sum','dram__bytes_write.sum','dram__cycles_active.avg.pct_of_peak_sustained_elapsed','sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active','lts__t_sector_hit_rate.pct','launch__registers_per_thread','l1tex__throughput.avg.pct_of_peak_sustained_elapsed','lts__throughput.avg.pct_of_peak_sustained_elapsed']:
    print(k, d.get(k), r[1][h.index(k)] if k in h else '')
P
rm -f gpurun_out/e_k1.ncu-rep
