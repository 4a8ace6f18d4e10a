cd scripts/umma
for N in 32 64 96 128 192 256; do for nacc in 1 2; do python run_probe.py rate 128 $N 32 148 $nacc; done; done
python run_probe.py rate 128 256 64 148 1
python run_probe.py rate 128 64 128 148 1
