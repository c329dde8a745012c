python tools/run_once.py C2
ncu --set full --import-source on --clock-control none -k regex:resident_kernel -c 1 -o gpurun_out/c2_res -f python tools/run_once.py C2 > gpurun_out/c2prof.log 2>&1; echo "ncu rc $?"
tail -2 gpurun_out/c2prof.log
