for B in 256 512; do python bench.py --no-cpu --config llama-3.1-8b --batch $B --steps 8 > gpurun_out/bench_llama_b$B.log 2>&1; done
