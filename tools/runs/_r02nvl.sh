set -u
out=gpurun_out/r02nvl
mkdir -p $out
export MASTER_ADDR=127.0.0.1 MASTER_PORT=29830 WORLD_SIZE=2 LARS_B200_LIB=liblars_b200.so
# the ncu wrapper runs rank 0 twice (once plain, once profiled): rank 1 partners both
( for i in 1 2; do RANK=1 LOCAL_RANK=1 timeout 200 python tools/trace_nvls.py --steps 8 > $out/r1_$i.log 2>&1; done ) &
RANK=0 LOCAL_RANK=0 timeout 450 ncu --metrics gpu__time_duration.sum,nvlrx__bytes.sum,nvltx__bytes.sum,nvlrx__bytes_data_user.sum,nvltx__bytes_data_user.sum,dram__bytes_read.sum,dram__bytes_write.sum \
  --clock-control none -k regex:lars_step_kernel --launch-skip 4 --launch-count 1 --csv --log-file $out/ncu_nvlink_p2.csv \
  python tools/trace_nvls.py --steps 8 > $out/r0.log 2>&1
echo "rank0 rc=$?"
wait
echo "rank1 done"
tail -12 $out/ncu_nvlink_p2.csv
