NLD_OZAKI=0 python scripts/oz_check.py c4 16 /tmp/a4.npy > /dev/null 2>&1
NLD_LIB=$PWD/paper_2407_06834_b200/libnld_b200_g1.so timeout 120 python scripts/oz_check.py c4 16 /tmp/b4.npy 2>&1 | tail -1
python scripts/oz_check.py cmp /tmp/b4.npy /tmp/a4.npy
bash scripts/ab.sh
