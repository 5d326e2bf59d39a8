for b in 6 8; do FSMC_DRAW_BLOCKS_PER_SM=$b timeout 300 python bench.py --draw-parts 2 --steps 3 --warmup 3 --no-cpu --no-lockstep > gpurun_out/r02_ovb_$b.json 2> gpurun_out/r02_ovb_$b.err; done
timeout 300 python bench.py --draw-parts 1 --steps 3 --warmup 3 --no-cpu --no-lockstep > gpurun_out/r02_ovb_p1.json 2> gpurun_out/r02_ovb_p1.err
