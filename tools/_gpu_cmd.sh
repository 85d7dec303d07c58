for v in t1024 t1024i1 t1024o4 t512m2 t256m4 t1024i1o8 t1024; do MLTUNE_B200_LIB=build/variants/$v/libmltune_b200.so python tools/sweep_ab.py synthetic-1e8 10; done > gpurun_out/tile_ab3.log 2>&1
for v in t1024 t1024o4; do MLTUNE_B200_LIB=build/variants/$v/libmltune_b200.so python tools/sweep_ab.py stereo 10; done >> gpurun_out/tile_ab3.log 2>&1
cat gpurun_out/tile_ab3.log
