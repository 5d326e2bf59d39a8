for w in 1100 3300 4096; do timeout 300 python bench.py --draw-window $w --steps 3 --warmup 3 --no-cpu --no-lockstep > gpurun_out/r02_w_$w.json 2> gpurun_out/r02_w_$w.err; done
