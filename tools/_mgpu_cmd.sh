make -s -C oracle >/dev/null 2>&1
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29533 bench.py --gpus 4 --steps 5 --warmup 3 > gpurun_out/bench_c3_n4_par.json 2> gpurun_out/bench_c3_n4_par.err
timeout 1500 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29534 bench.py --config c4 --gpus 4 --steps 3 --warmup 3 --parity-rows 3 > gpurun_out/bench_c4_n4_par.json 2> gpurun_out/bench_c4_n4_par.err
for f in gpurun_out/bench_c3_n4_par.json gpurun_out/bench_c4_n4_par.json; do tail -c 700 $f; echo; done
grep -v "^\*\|OMP" gpurun_out/bench_c4_n4_par.err | tail -5
