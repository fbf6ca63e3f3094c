# Process start-up variance on the GPU box: persistence mode, and the CUDA init time of
# 8 back-to-back fresh processes without and with a process holding a CUDA context.
nvidia-smi -q | grep -i -A1 "persistence"
cat > /tmp/ci.py <<'PY'
import ctypes, time
t=time.perf_counter(); lib=ctypes.CDLL("libcudart.so.12") if False else None
PY
cat > /tmp/ci.c <<'C'
#include <cuda_runtime.h>
#include <stdio.h>
#include <time.h>
int main(){struct timespec a,b;clock_gettime(CLOCK_MONOTONIC,&a);int n=0;cudaGetDeviceCount(&n);cudaFree(0);clock_gettime(CLOCK_MONOTONIC,&b);printf("%.3f\n",(b.tv_sec-a.tv_sec)+1e-9*(b.tv_nsec-a.tv_nsec));return 0;}
C
nvcc -o /tmp/ci /tmp/ci.c
echo "no keeper:"; for i in 1 2 3 4 5 6 7 8; do /tmp/ci; sleep 0.3; done | tr '\n' ' '; echo
cat > /tmp/keep.c <<'C'
#include <cuda_runtime.h>
#include <unistd.h>
int main(){cudaFree(0);for(;;) pause();}
C
nvcc -o /tmp/keep /tmp/keep.c; /tmp/keep & K=$!; sleep 2
echo "keeper:"; for i in 1 2 3 4 5 6 7 8; do /tmp/ci; sleep 0.3; done | tr '\n' ' '; echo
kill $K
