S1=$PWD/paper_2207_01205_b200/_lib/libfofse_s1.so
FOFSE_LIB_PATH=$S1 timeout 600 python tools/parity_study_batch.py C3 1 300 4:1e-5 2>&1 | tail -1
timeout 600 python tools/parity_study_batch.py C3 1 300 4:1e-5 2>&1 | tail -1
FOFSE_CHUNK_MIN=24576 timeout 600 python tools/parity_study_batch.py C3 1 300 4:1e-5 2>&1 | tail -1
FOFSE_HEAD_TM=1 timeout 600 python tools/parity_study_batch.py C3 1 300 4:1e-5 2>&1 | tail -1
FOFSE_LIB_PATH=$S1 timeout 600 python tools/parity_study_batch.py C3 4 300 4:1e-5 2>&1 | tail -1
