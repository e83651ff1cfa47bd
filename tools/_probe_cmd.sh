make -s -C oracle >/dev/null 2>&1
timeout 300 python -m pytest tests/test_gpu_parity.py -q -k "pipelined or batch_of or streamed or streaming or tensor_core" 2>&1 | tail -2
for r in 1 2 3; do for v in "--define TF_TC_NOPROBE" "--define TF_TC_NOPROBE --define TF_TC_FLUSH2"; do timeout 60 python tools/tc_probe.py --n 2048 --n-proj 1800 --rows 1024 --reps 2 $v 2>&1 | tail -1; done; done
timeout 900 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-parity > gpurun_out/bench_e2e2.json 2>&1
python -c "import json; d=json.loads(open('gpurun_out/bench_e2e2.json').read().strip().splitlines()[-1]); print(d['s_per_volume'], d['e2e']['s_per_volume'], d['e2e']['vs_device_resident'], d['e2e']['matches_device_resident_volume_bitwise'], d['clocks'])"
