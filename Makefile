# Builds libmpsf.so (sm_100a only) and the C oracle.  __graft_entry__.build() runs the same.
NVCC ?= nvcc
ARCH := -gencode arch=compute_100a,code=sm_100a
NVFLAGS := -O3 -lineinfo -std=c++17 $(ARCH) -Xcompiler -fPIC,-O3 -Iinclude -Xptxas -v
SRC := $(wildcard paper_2605_26461_b200/csrc/*.cu paper_2605_26461_b200/csrc/*.cpp)
HDR := $(wildcard paper_2605_26461_b200/csrc/*.cuh paper_2605_26461_b200/csrc/*.h) include/mpsf.h

all: paper_2605_26461_b200/libmpsf.so

paper_2605_26461_b200/libmpsf.so: $(SRC) $(HDR)
	$(NVCC) $(NVFLAGS) -shared -o $@ $(SRC) 2> build_ptxas.log || (cat build_ptxas.log; false)

clean:
	rm -f paper_2605_26461_b200/libmpsf.so build_ptxas.log
