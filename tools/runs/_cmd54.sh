bash tools/ab_build.sh base "" nommas "-DS2L_EXP_NO_S -DS2L_EXP_NO_PV -DS2L_SPLIT_S=0" nosplit "-DS2L_SPLIT_S=0"
