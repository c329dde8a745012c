ncu --metrics gpu__time_duration.sum --clock-control none --kernel-name-base demangled -k regex:aw:: -c 400 --csv --log-file gpurun_out/launches_C3_r2.csv \
    python bench.py --steps 1 --warmup 3 --nt 50 --no-cpu-baseline --no-e2e > gpurun_out/ncu_ll.log 2>&1; echo "launch list rc $?"
