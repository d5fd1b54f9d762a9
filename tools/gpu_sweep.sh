for B in 32 128 256; do python bench.py --no-cpu --batch $B --steps 10 > gpurun_out/bench_b$B.log 2>&1; done
for B in 64 256; do python bench.py --no-cpu --config llama-3.1-8b --batch $B --steps 10 > gpurun_out/bench_llama_b$B.log 2>&1; done
