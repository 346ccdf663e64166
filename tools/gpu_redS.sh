for S in 16 8 4 2; do echo "S=$S"; NB_RED_SLICES=$S timeout 120 python tools/trainbench.py c2 200; NB_RED_SLICES=$S timeout 120 python tools/trainbench.py c3 200; done
