for gr in 0 8 16 32 64 148; do
  if [ $gr = 0 ]; then python tools/chol_grid.py; else RLRA_CHOL_GRID=$gr python tools/chol_grid.py; fi
done
