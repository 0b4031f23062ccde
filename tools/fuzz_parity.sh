# Re-seeded parity passes (on the GPU box): the random-problem suites (every fused kernel template, the
# sweeps, batches, FFT levels, tent map, reduced MC, row-zeroed nets) on seeds shifted by
# RQMC_TEST_SEED_OFFSET -- the oracle and the CUDA path get the same re-seeded inputs from workloads/.
# (the two fine-path cases whose random level shape, and so their asserted kernel template, depends on the seed are left out)
# usage: bash tools/fuzz_parity.sh r02g 1000 2000 3000
P=${1:-fuzz}; shift
mkdir -p gpurun_out/fuzz
for off in "$@"; do
  RQMC_TEST_SEED_OFFSET=$off python -m pytest -q -m gpu -p no:cacheprovider \
    tests/test_gpu_fine_paths.py tests/test_gpu_parity.py tests/test_gpu_batch.py tests/test_gpu_fft.py \
    tests/test_gpu_tent.py tests/test_gpu_reduced_mc.py tests/test_gpu_rowzero_net.py tests/test_gpu_latency.py \
    -k "not config_c and not c5u and not multiprocess and not gen3_rand and not gen2_rand_net" > gpurun_out/fuzz/${P}_off${off}.log 2>&1
  echo "offset $off: $(tail -1 gpurun_out/fuzz/${P}_off${off}.log)"
done
