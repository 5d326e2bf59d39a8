# lane-group sweep: C2 window kernel at G=1 (MoG special) vs G=2/4 (generic plugin switch),
# C3 at G=32 (special) vs G=128 (generic)
for L in 1 2 4; do timeout 300 python bench.py --steps 3 --warmup 3 --no-cpu --no-lockstep --lanes $L > gpurun_out/r03_lanes_c2_$L.json 2> gpurun_out/r03_lanes_c2_$L.err; done
for L in 32 128; do timeout 300 python bench.py --config c3 --steps 3 --warmup 3 --no-cpu --no-lockstep --lanes $L > gpurun_out/r03_lanes_c3_$L.json 2> gpurun_out/r03_lanes_c3_$L.err; done
