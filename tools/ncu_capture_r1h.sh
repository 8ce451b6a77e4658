set -x
mkdir -p gpurun_out/h
K1='regex:.*RegionsProg.*'; K2='regex:.*SharedArrayProg.*'; K3='regex:.*NestedProg.*'; K4='regex:.*StreamProg.*'
ncu --set full --import-source on --clock-control none --kernel-name-base mangled -k "$K1" -s 1 -c 1 -o gpurun_out/h/regions -f python tools/regions_long_probe.py > gpurun_out/h/regions.log 2>&1
ncu --set full --import-source on --clock-control none --kernel-name-base mangled -k "$K2" -s 1 -c 1 -o gpurun_out/h/config2 -f python tools/config2_probe.py > gpurun_out/h/config2.log 2>&1
ncu --set full --import-source on --clock-control none --kernel-name-base mangled -k "$K3" -s 1 -c 1 -o gpurun_out/h/nested -f python tools/nested_full_probe.py > gpurun_out/h/nested.log 2>&1
ncu --set full --import-source on --clock-control none --kernel-name-base mangled -k "$K4" -s 2 -c 1 -o gpurun_out/h/stream -f python bench.py --steps 3 --warmup 3 > gpurun_out/h/stream.log 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none -c 600 --csv --log-file gpurun_out/h/launches.csv python bench.py --steps 20 --warmup 3 > gpurun_out/h/launch_bench.log 2>&1
ls -la gpurun_out/h
