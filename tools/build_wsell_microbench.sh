# the microbenchmark with its own copy of engine.cpp (the host layout builder must be
# compiled with the same F3RG_WS_* defines as the kernels); everything else from libf3rg.so
set -e
cd "$(dirname "$0")/.."
g++ -std=c++17 -O2 -fPIC -ffp-contract=off -I/usr/local/cuda/include -Wall -Wno-unused -fopenmp $WSDEFS -c paper_2505_20719_b200/csrc/engine.cpp -o build/engine${WSNAME}.o
nvcc -std=c++17 -O3 -lineinfo -fmad=false -gencode arch=compute_100a,code=sm_100a --expt-relaxed-constexpr -Xptxas -v $WSDEFS -I paper_2505_20719_b200/csrc tools/wsell_microbench.cu build/engine${WSNAME}.o -o build/wsell_microbench${WSNAME} -Xcompiler -fopenmp -L paper_2505_20719_b200/lib -lf3rg -Xlinker -rpath -Xlinker '$ORIGIN/../paper_2505_20719_b200/lib' 2>&1 | grep -E "error|warning|kb_|registers|spill" | grep -v "k_fill"
