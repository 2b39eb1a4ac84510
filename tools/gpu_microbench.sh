mkdir -p gpurun_out
./tools/microbench/mailbox_lat > gpurun_out/mailbox_lat.txt 2>&1
./tools/microbench/sync_lat > gpurun_out/sync_lat.txt 2>&1
echo done
