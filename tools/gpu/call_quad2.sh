bash tools/gpu/ab.sh quad6 "FOFSE_V2R_VAR=0" "FOFSE_V2R_VAR=6" 2
