for i in 1 2; do
  for v in hbm smem; do
    for w in "api64 100000" "chat1024 30000" "agent256 10000" "cfg1 10000"; do
      set -- $w
      if [ $v = hbm ]; then export RSIM_NO_SMEM_RUNNING=1; else unset RSIM_NO_SMEM_RUNNING; fi
      timeout 200 python tools/profile_replay.py $1 $2 2>&1 | grep "us/decision" | sed "s/^/[$v] /"
    done
  done
done
