for n in scn_table4_obstacles_1000_5x syn_se2_m80; do
python tools/gpu/bisect.py $n
RGG_GPU_LIB=tools/gpu/lib_head/librgg_gpu.so python tools/gpu/bisect.py $n
RGG_EARLY_TOUCH_MIN=100000 python tools/gpu/bisect.py $n
RGG_NO_EARLY_BIN=1 python tools/gpu/bisect.py $n
RGG_NO_GRAPH=1 python tools/gpu/bisect.py $n
done
