set -x
python tools/ab_c2svd.py
python tools/ab_c2svd.py tools/_ab/librlra_b200_nopair.so
