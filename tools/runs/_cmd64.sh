timeout -s KILL 300 python tools/fused_diag.py ab_libs/new2.so ab_libs/new2.so:FUSED=1 ab_libs/nowrite.so:FUSED=1 ab_libs/poolread.so:FUSED=1 8
timeout -s KILL 300 python tools/fused_diag.py ab_libs/poolread.so:FUSED=1 ab_libs/nowrite.so:FUSED=1 ab_libs/new2.so:FUSED=1 ab_libs/new2.so 8
