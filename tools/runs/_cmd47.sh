bash tools/ab_build.sh base "" hsplit_p2 "-DS2L_HSPLIT=1 -DS2L_POLY_PAIRS=2" hsplit_p4 "-DS2L_HSPLIT=1 -DS2L_POLY_PAIRS=4" base_p2 "-DS2L_POLY_PAIRS=2"
