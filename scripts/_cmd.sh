python scripts/oz_check.py c1 16 /tmp/a1.npy 2>&1 | tail -1
NLD_OZAKI=1 timeout 120 python scripts/oz_check.py c1 16 /tmp/b1.npy 2>&1 | tail -3
python scripts/oz_check.py cmp /tmp/b1.npy /tmp/a1.npy
python scripts/oz_check.py c4 16 /tmp/a4.npy 2>&1 | tail -1
NLD_OZAKI=1 timeout 120 python scripts/oz_check.py c4 16 /tmp/b4.npy 2>&1 | tail -3
python scripts/oz_check.py cmp /tmp/b4.npy /tmp/a4.npy
NLD_OZAKI=1 bash scripts/ab_env.sh oz "X=0"
