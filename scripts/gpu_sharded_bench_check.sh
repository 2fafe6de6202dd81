# The multi-GPU bench path end to end on a one-GPU box: two ranks pinned to
# cuda:0 exchanging over gloo (validation of the sharded plumbing only; the
# driver's multi-GPU runs use one GPU per rank and NCCL)
MARS_DEBUG_LAUNCH=1 MARS_BENCH_DEVICE=0 MARS_BENCH_BACKEND=gloo timeout 600 \
  python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 \
  --master-port 29533 bench.py --gpus 2 --steps 3 --warmup 3 --no-kv --hbm-sweep "" \
  --e2e-steps 1 --sessions 200000 > gpurun_out/sharded2.json 2> gpurun_out/sharded2.err
echo "rc=$?"
tail -c 400 gpurun_out/sharded2.json
grep "mars:" gpurun_out/sharded2.err | head
