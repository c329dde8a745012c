timeout 600 python -m pytest tests/test_gpu_boundary.py tests/test_gpu_resident2d.py -x -q 2>&1 | tail -2
ncu --metrics gpu__time_duration.sum --clock-control none --kernel-name-base demangled -k regex:stage_model -c 4 --csv \
    python bench.py --steps 1 --warmup 3 --nt 5 --no-cpu-baseline --no-e2e 2>/dev/null | grep stage_model | awk -F'","' '{print $NF}'
