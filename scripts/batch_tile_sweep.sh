for W in 16 8; do for SP in 0 1; do
  echo "W=$W split=$SP" >> gpurun_out/sw.log
  HELM_BATCH_W=$W HELM_BATCH_SPLIT=$SP timeout 300 python scripts/shard_timing.py c3 1,2,4,8 2>&1 | grep -v "N=1 apply" >> gpurun_out/sw.log
done; done
