for b in 1 2 3 4 6 8 16; do echo "BE=$b"; HP_FG_BLOCK=$b python tools/time_matvec.py cfg4; done
