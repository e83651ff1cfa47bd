make -s -C oracle >/dev/null 2>&1
timeout 300 python -m pytest tests/test_gpu_parity.py -q -k "batch_of_specimens or streaming" 2>&1 | tail -3
timeout 1200 python bench.py --config c5 --rows 256 --slab-rows 128 --specimens 2 --steps 2 --warmup 1 > gpurun_out/bench_c5_stream.json 2> gpurun_out/bench_c5_stream.err; tail -c 1800 gpurun_out/bench_c5_stream.json; tail -2 gpurun_out/bench_c5_stream.err
timeout 900 python bench.py --config c4 --rows 512 --slab-rows 256 --specimens 2 --steps 2 --warmup 1 > gpurun_out/bench_c4_stream.json 2> gpurun_out/bench_c4_stream.err; tail -c 1800 gpurun_out/bench_c4_stream.json; tail -2 gpurun_out/bench_c4_stream.err
