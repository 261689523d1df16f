cd /root/repo
for sh in "0 0" "15 3" "8 4" "8 8" "11 3" "15 2" "4 8" "6 6"; do
  timeout 200 python tools/profile_replay.py api64 100234 $sh 2>&1 | grep "us/decision" | sed "s/total [0-9.]* ms  replay [0-9.]* ms//"
done
for sh in "0 0" "15 7" "12 7" "15 5" "10 7"; do
  timeout 200 python tools/profile_replay.py chat1024 40000 $sh 2>&1 | grep "us/decision" | sed "s/total [0-9.]* ms  replay [0-9.]* ms//"
done
