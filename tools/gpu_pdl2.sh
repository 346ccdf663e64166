# PDL across the non-fused training chain: timing + training tests
mkdir -p gpurun_out
for r in 1 2; do for c in c2 c3 c4 c5; do timeout 120 python tools/trainbench.py $c 200; done; done
timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_depth.py tests/test_hierarchy.py -x -q -p no:cacheprovider -k "train or grad or adam or micro or graph or control or two_shards or sine or pe or schedule or stats or loss or hier" > gpurun_out/pdl2_tests.log 2>&1; echo "rc=$?" >> gpurun_out/pdl2_tests.log
tail -n 3 gpurun_out/pdl2_tests.log
