mkdir -p gpurun_out
for b in 1 16 64; do
  for be in split chain; do
    echo "== B=$b backend=$be"
    timeout 300 python tools/attrib.py --batch $b --mlp-backend $be --only "mlp(up+down)"
  done
done > gpurun_out/attrib_mlp.log 2>&1
