T=gpurun_out/r02ae; mkdir -p $T
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/random_probe tools/probe/random_probe.cu && /tmp/random_probe > $T/random_probe.json 2>&1; echo "rc=$?"; cat $T/random_probe.json
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/stream_probe tools/probe/stream_probe.cu && /tmp/stream_probe > $T/stream_probe.txt 2>&1; cat $T/stream_probe.txt
