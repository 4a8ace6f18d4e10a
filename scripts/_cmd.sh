NLD_OZAKI=0 python scripts/oz_check.py c4 16 /tmp/a4.npy > /dev/null 2>&1
timeout 120 python scripts/oz_check.py c4 16 /tmp/b4.npy 2>&1 | tail -1
python scripts/oz_check.py cmp /tmp/b4.npy /tmp/a4.npy
bash scripts/ab_env.sh persist X=0 nopersist NLD_GATHER_PERSIST=0
timeout 600 python scripts/shard_probe.py 2>&1 | grep shard
