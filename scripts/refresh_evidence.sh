set -x
mkdir -p gpurun_out/rf
timeout 900 python -m pytest -q tests -m gpu > gpurun_out/rf/pytest_gpu.txt 2>&1; tail -2 gpurun_out/rf/pytest_gpu.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/rf/smoke.txt 2>&1; tail -1 gpurun_out/rf/smoke.txt
for w in resnet18 resnet18_ma resnet18_4w resnet50 resnet50_3w mlp; do
  timeout 500 python bench.py --workload $w > gpurun_out/rf/bench_$w.json 2> gpurun_out/rf/bench_$w.err; tail -c 200 gpurun_out/rf/bench_$w.json; echo
done
timeout 120 python scripts/time_convs.py r18 step > gpurun_out/rf/conv_times_r18.txt 2>&1
timeout 120 python scripts/time_convs.py r50 step > gpurun_out/rf/conv_times_r50.txt 2>&1
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -s 240 -c 400 --csv --log-file gpurun_out/rf/launches_step.csv python scripts/ncu_step.py step > /dev/null 2>&1
timeout 300 ncu --set full --import-source on --clock-control none -k regex:gemm_bf16 -s 2 -c 1 -o gpurun_out/rf/wgrad64 python scripts/ncu_conv.py 128 32 64 64 3 1 wgrad 4 > /dev/null 2>&1
timeout 300 ncu --set full --import-source on --clock-control none -k regex:gemm_bf16 -s 2 -c 1 -o gpurun_out/rf/dgrad128 python scripts/ncu_conv.py 128 16 128 128 3 1 dgrad 4 > /dev/null 2>&1
timeout 300 ncu --set full --import-source on --clock-control none -k regex:gemm_bf16 -s 2 -c 1 -o gpurun_out/rf/halo64 python scripts/ncu_conv.py 128 32 64 64 3 1 fwd 4 > /dev/null 2>&1
ls -la gpurun_out/rf
