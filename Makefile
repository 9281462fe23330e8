# Product build: libfw2v.so (C-ABI + sm_100a kernels) and the ringvec::train
# drop-in shim, both in-tree under paper_2312_07743_b200/_lib/ so they travel
# to the GPU box with the gpurun snapshot. `make oracle` builds the checkers
# (oracle/Makefile); `make all` does both plus the reference suites linked
# against the drop-in.

NVCC     ?= /usr/local/cuda/bin/nvcc
CXX      ?= g++
ARCH     := -gencode arch=compute_100a,code=sm_100a
PKG      := paper_2312_07743_b200
SRC      := $(PKG)/csrc
LIB      := $(PKG)/_lib
BUILD    := build
REF      ?= /root/reference/proj
CUDA_INC := /usr/local/cuda/include

NVFLAGS  := -O3 -std=c++17 $(ARCH) -lineinfo -Xcompiler -fPIC -Xptxas -v -Iinclude -I$(SRC)
CXXFLAGS := -O2 -std=c++17 -fPIC -Wall -Wextra -Iinclude -I$(SRC) -I$(CUDA_INC)

.PHONY: all lib dropin oracle suite clean
all: lib dropin oracle suite

lib: $(LIB)/libfw2v.so

$(BUILD)/fw2v_kernels.o: $(SRC)/fw2v_kernels.cu $(SRC)/fw2v_device.cuh
	@mkdir -p $(BUILD)
	$(NVCC) $(NVFLAGS) -c -o $@ $< 2> $(BUILD)/ptxas_kernels.log || (cat $(BUILD)/ptxas_kernels.log; false)

$(BUILD)/fw2v_snapshot.o: $(SRC)/fw2v_snapshot.cu $(SRC)/fw2v_device.cuh $(SRC)/fw2v_common.cuh
	@mkdir -p $(BUILD)
	$(NVCC) $(NVFLAGS) -c -o $@ $< 2> $(BUILD)/ptxas_snapshot.log || (cat $(BUILD)/ptxas_snapshot.log; false)

$(BUILD)/fw2v_host.o: $(SRC)/fw2v_host.cpp include/fw2v.h $(SRC)/fw2v_device.cuh
	@mkdir -p $(BUILD)
	$(CXX) $(CXXFLAGS) -c -o $@ $<

$(BUILD)/fw2v_corpus.o: $(SRC)/fw2v_corpus.cpp include/fw2v.h
	@mkdir -p $(BUILD)
	$(CXX) $(CXXFLAGS) -O3 -c -o $@ $<

$(LIB)/libfw2v.so: $(BUILD)/fw2v_kernels.o $(BUILD)/fw2v_snapshot.o $(BUILD)/fw2v_host.o $(BUILD)/fw2v_corpus.o
	@mkdir -p $(LIB)
	$(NVCC) $(ARCH) -shared -cudart static -o $@ $^ -lpthread -ldl -lrt

# ringvec::train drop-in, compiled against the reference's public headers.
dropin: $(LIB)/libringvec_fw2v.so

$(LIB)/libringvec_fw2v.so: $(SRC)/ringvec_train_fw2v.cpp $(LIB)/libfw2v.so include/fw2v.h
	@if [ -d $(REF)/include ]; then \
	  $(CXX) -std=c++20 -O2 -fPIC -shared -Iinclude -I$(REF)/include -o $@ $< \
	    -L$(LIB) -lfw2v -Wl,-rpath,'$$ORIGIN'; \
	else echo "reference headers absent: keeping prebuilt $@"; fi

oracle:
	$(MAKE) -C oracle all

suite: dropin
	$(MAKE) -C oracle gpu-suite

clean:
	rm -rf $(BUILD) $(LIB)
