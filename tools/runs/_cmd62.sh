timeout -s KILL 600 python tools/ab.py ab_libs/head.so ab_libs/new.so ab_libs/new.so:FUSED=1 8
timeout -s KILL 600 python tools/ab.py ab_libs/new.so:FUSED=1 ab_libs/new.so ab_libs/head.so 8
