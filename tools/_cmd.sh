make -s -C oracle >/dev/null 2>&1
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" 2>&1 | tail -2
timeout 900 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err; tail -c 800 gpurun_out/bench_ref.json; echo
timeout 1500 python bench.py --steps 10 --warmup 3 > gpurun_out/bench_final.json 2> gpurun_out/bench_final.err
python - <<'P'
import json
d=json.loads(open('gpurun_out/bench_final.json').read().strip().splitlines()[-1])
print(d['value'], d['s_per_volume'], d['e2e']['s_per_volume'], d['e2e']['matches_device_resident_volume_bitwise'], d['clocks'])
print(d['roofline']['frac'], d['roofline']['tensor_pipe']['frac'], d['cpu_baseline']['value'], d['parity']['rel_l2_vs_f64_oracle'], d['gpu_launches'])
P
tail -3 gpurun_out/bench_final.err
