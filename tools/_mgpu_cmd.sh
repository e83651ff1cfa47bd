make -s -C oracle >/dev/null 2>&1
python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29601 tools/host_link.py 2>/dev/null | tail -1 > gpurun_out/hostlink_n1.json
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29602 bench.py --gpus 4 --steps 10 --warmup 3 > gpurun_out/bench_c3_n4.json 2> gpurun_out/bench_c3_n4.err
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29603 bench.py --gpus 2 --steps 10 --warmup 3 > gpurun_out/bench_c3_n2.json 2> gpurun_out/bench_c3_n2.err
timeout 1200 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29604 bench.py --gpus 4 --config c4 --steps 3 --warmup 2 > gpurun_out/bench_c4_n4.json 2> gpurun_out/bench_c4_n4.err
for f in hostlink_n1 bench_c3_n4 bench_c3_n2 bench_c4_n4; do echo "== $f"; tail -c 1500 gpurun_out/$f.json; done
tail -3 gpurun_out/bench_c4_n4.err
