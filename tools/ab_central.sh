cd /root/repo
for pass in 1 2; do for w in "api64 100234" "chat1024 40000" "agent256 8000" "large4096 60000" "chat16 10000"; do
  RSIM_NO_CENTRAL=1 timeout 200 python tools/profile_replay.py $w 2>&1 | grep "us/decision" | sed "s/ctas=0 warps=0: total [0-9.]* ms  replay [0-9.]* ms//; s/^/[old p$pass] /"
  timeout 200 python tools/profile_replay.py $w 2>&1 | grep "us/decision" | sed "s/ctas=0 warps=0: total [0-9.]* ms  replay [0-9.]* ms//; s/^/[central p$pass] /"
done; done
