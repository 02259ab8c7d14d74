for N in 4 2; do
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port $((29500 + RANDOM % 1000)) tools/dist_parity.py > gpurun_out/dp2_$N.log 2>&1; echo "N=$N parity rc=$?"; grep -E "^(OK|BAD)" gpurun_out/dp2_$N.log | grep -c OK; grep -E "^BAD|golden" gpurun_out/dp2_$N.log
done
bash tools/multi_r2.sh 4 2>&1 | grep -A1 devloop
