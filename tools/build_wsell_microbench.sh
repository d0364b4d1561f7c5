# microbenchmark of the windowed engine without the 10-minute library build: recompiles only
# engine.cpp and launch_setup.cu (the layout side), relinks libf3rg.so from the existing objects
# (the other objects may be stale -- run ONLY the microbenchmark against this library), then the tool
set -e
cd "$(dirname "$0")/.."
g++ -std=c++17 -O2 -fPIC -ffp-contract=off -I/usr/local/cuda/include -Wall -Wno-unused -fopenmp $WSDEFS -c paper_2505_20719_b200/csrc/engine.cpp -o build/obj/engine.cpp.o
nvcc -std=c++17 -O3 -lineinfo -fmad=false -gencode arch=compute_100a,code=sm_100a -Xcompiler -fPIC --expt-relaxed-constexpr $WSDEFS -c paper_2505_20719_b200/csrc/launch_setup.cu -o build/obj/launch_setup.cu.o
g++ -shared -o paper_2505_20719_b200/lib/libf3rg.so build/obj/*.o -L/usr/local/cuda/lib64 -lcudart_static -ldl -lrt -lpthread -fopenmp -L/usr/lib/x86_64-linux-gnu -l:libstdc++.so.6 -Wl,-soname,libf3rg.so -Wl,--no-undefined
nvcc -std=c++17 -O3 -lineinfo -fmad=false -gencode arch=compute_100a,code=sm_100a --expt-relaxed-constexpr -Xptxas -v $WSDEFS -I paper_2505_20719_b200/csrc tools/wsell_microbench.cu -o build/wsell_microbench${WSNAME} -L paper_2505_20719_b200/lib -lf3rg -Xlinker -rpath -Xlinker '$ORIGIN/../paper_2505_20719_b200/lib' 2>&1 | grep -E "error|warning|kb_|registers|spill" | grep -v "k_fill"
