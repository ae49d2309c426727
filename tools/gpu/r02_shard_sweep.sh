mkdir -p gpurun_out/sweep; O=gpurun_out/sweep
for cfg in c3 c2_bf16; do
  python tools/shard_time.py $cfg > $O/${cfg}_base.log 2>&1
  LRS_WCONV_IPW=4 python tools/shard_time.py $cfg > $O/${cfg}_ipw4.log 2>&1
  LRS_WCONV_CB=2 python tools/shard_time.py $cfg > $O/${cfg}_cb2.log 2>&1
  LRS_WCONV_TH=1 python tools/shard_time.py $cfg > $O/${cfg}_th1.log 2>&1
  LRS_WCONV_IPW=4 LRS_WCONV_TH=1 python tools/shard_time.py $cfg > $O/${cfg}_ipw4_th1.log 2>&1
done
