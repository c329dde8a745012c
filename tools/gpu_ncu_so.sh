# GPU box: one `ncu --set full` capture (with source) of the 3D streaming kernel at space order $SO on 512^3
SO=${SO:-16}
timeout 900 ncu --set full --import-source on --clock-control none -k regex:stream_kernel --launch-skip 12 -c 1 \
  -o gpurun_out/stream_so${SO} -f python tools/ab_stream.py --child ${SO} --nt 10 > gpurun_out/ncu_so${SO}.log 2>&1
tail -3 gpurun_out/ncu_so${SO}.log
