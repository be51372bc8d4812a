bash tools/ab_build.sh split "" nosplit "-DS2L_SPLIT_S=0" nosplit_p2 "-DS2L_SPLIT_S=0 -DS2L_POLY_PAIRS=2" nosplit_nosm64 "-DS2L_SPLIT_S=0 -DS2L_SM64=0"
