S2L_EXP_BOX_ROWS=32 bash tools/exp_variants.sh "-DS2L_EXP_MMA_ONLY -DS2L_EXP_NO_S -DS2L_EXP_NO_PV -DS2L_EXP_BOX32"
bash tools/exp_variants.sh "-DS2L_EXP_MMA_ONLY -DS2L_EXP_NO_S -DS2L_EXP_NO_PV"
