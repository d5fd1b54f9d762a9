mkdir -p gpurun_out
timeout 200 python -m pytest tests/test_gpu_chain.py -x -q > gpurun_out/chain.log 2>&1
for b in 1 64 256; do timeout 60 python tools/chain_trace.py $b; done > gpurun_out/chain_trace.log 2>&1
timeout 240 python tools/chain_bench.py --router ${CB_ARGS:-} > gpurun_out/chain_bench.log 2>&1
for b in 1 16 64; do
  for be in split chain; do
    echo "== B=$b backend=$be"
    timeout 300 python tools/attrib.py --batch $b --mlp-backend $be --only "mlp(up+down)"
  done
done > gpurun_out/attrib_mlp.log 2>&1
