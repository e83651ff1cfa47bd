timeout 1500 python bench.py --config c5 --steps 1 --warmup 1 --rows 256 --slab-rows 256 --specimens 2 > gpurun_out/bench_c5_chunked.json 2> gpurun_out/bench_c5_chunked.err
for f in gpurun_out/bench_c5_chunked.json; do python -c "
import json,sys; d=json.loads(open('$f').read().strip().splitlines()[-1]); print(d['value'], d['ms_per_step'], d['config']['angle_chunk'], d['config']['device_free_gb_at_setup'], d['clocks'])"; done
tail -3 gpurun_out/bench_c5_chunked.err
