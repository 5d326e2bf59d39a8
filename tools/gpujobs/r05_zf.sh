# row-reuse race evidence: the new stress test on HEAD (must pass) and on the pre-fix read-back build (expected to fail)
mkdir -p gpurun_out/r05zf
timeout 900 python -m pytest tests/test_gpu_parity.py -q -p no:cacheprovider -k "row_reuse_race" > gpurun_out/r05zf/head.log 2>&1; tail -2 gpurun_out/r05zf/head.log
FSMC_LIB=$(realpath variants/readback2/libfsmc.so) timeout 900 python -m pytest tests/test_gpu_parity.py -q -p no:cacheprovider -k "batched_evaluation_rounds_have_no_row_reuse_race" > gpurun_out/r05zf/readback.log 2>&1; tail -4 gpurun_out/r05zf/readback.log
