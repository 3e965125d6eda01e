mkdir -p gpurun_out
RF_LIB_PATH=$PWD/variants/lib_tma.so timeout 600 python -m pytest tests/test_volume_gpu.py tests/test_edge_cases_gpu.py tests/test_reintegration.py -m gpu -q -x 2>&1 | tail -3 > gpurun_out/tma_tests.log
timeout 300 python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-e2e > /dev/null 2>&1
STEPS=8 bash tools/ab_bench.sh > gpurun_out/ab1.txt 2>&1
STEPS=8 bash tools/ab_bench.sh > gpurun_out/ab1b.txt 2>&1
timeout 300 python tools/bench_fusion.py > gpurun_out/fusion2.json 2> gpurun_out/fusion2.err
for v in base tma; do
RF_LIB_PATH=$PWD/variants/lib_$v.so timeout 600 ncu --set full --clock-control none --import-source on -k regex:"k_fuse" -s 20 -c 3 -o gpurun_out/prof_ab_$v python tools/prof_workload.py --build 20 --corrections 1 > /dev/null 2>&1
done
