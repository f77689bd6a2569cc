for c in c3:64 c3:1 c5:1 c5:8 c5:32 c2:16 c1:1; do python tools/fine_sweep.py --cases $c; done
