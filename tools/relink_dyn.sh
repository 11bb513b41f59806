cd paper_1905_08375_b200/_lib
OBJS=$(ls obj/*.o)
/usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -shared -o libnlgpu.so $OBJS -cudart shared -L/usr/local/cuda/lib64 -lcufft -Xlinker -rpath=/usr/local/cuda/lib64 -lrt -ldl -lpthread
cd ../..
ldd paper_1905_08375_b200/_lib/libnlgpu.so | grep -E "cudart|cufft"
python tools/dbg_es5.py 65536 00
