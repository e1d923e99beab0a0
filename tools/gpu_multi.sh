# bench code-path checks: 2 ranks sharing one GPU over gloo, and the reference arm on a small N
mkdir -p gpurun_out
SKEL_DIST_BACKEND=gloo timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29517 bench.py --gpus 2 --steps 2 --warmup 1 --points 262144 --nrhs-big 64 > gpurun_out/bench_2rank_gloo.log 2>&1; echo "2-rank rc=$?"; tail -1 gpurun_out/bench_2rank_gloo.log | cut -c1-600
timeout 600 python bench.py --impl reference --steps 1 --warmup 0 --points 65536 > gpurun_out/bench_ref_small.log 2>&1; echo "ref rc=$?"; tail -1 gpurun_out/bench_ref_small.log | cut -c1-400
