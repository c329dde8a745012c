python tools/run_once.py C1
ncu --set full --import-source on --clock-control none -k regex:resident2d -c 1 -o gpurun_out/c1_res2d -f python tools/run_once.py C1 > gpurun_out/c1prof.log 2>&1; echo "ncu rc $?"
tail -3 gpurun_out/c1prof.log
