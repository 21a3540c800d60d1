bash tools/gpu/abn.sh s3b 2 FOFSE_AB=base FOFSE_V2C_COPIES=2 FOFSE_V2C_COPIES=1
