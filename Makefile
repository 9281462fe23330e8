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

.PHONY: all lib dropin harness oracle suite clean
all: lib dropin harness oracle suite

lib: $(LIB)/libfw2v.so

$(BUILD)/fw2v_kernels.o: $(SRC)/fw2v_kernels.cu $(SRC)/fw2v_device.cuh
	@mkdir -p $(BUILD)
	$(NVCC) $(NVFLAGS) -c -o $@ $< 2> $(BUILD)/ptxas_kernels.log || (cat $(BUILD)/ptxas_kernels.log; false)

# K1s: one translation unit per lane shape (compiled in parallel), plus the dispatch.
K1S_SHAPES := l4v4 l8v4 l16v4 l16v8 l32v4 l32v6 l32v8 l32v10 l32v12 l32v16 l64v8
K1S_OBJS   := $(addprefix $(BUILD)/k1s_,$(addsuffix .o,$(K1S_SHAPES)))
K1S_DEPS   := $(SRC)/fw2v_snapshot.cuh $(SRC)/fw2v_stair.cuh $(SRC)/fw2v_device.cuh $(SRC)/fw2v_common.cuh

$(BUILD)/k1s_%.o: $(SRC)/k1s_%.cu $(K1S_DEPS)
	@mkdir -p $(BUILD)
	$(NVCC) $(NVFLAGS) -c -o $@ $< 2> $(BUILD)/ptxas_k1s_$*.log || (cat $(BUILD)/ptxas_k1s_$*.log; false)

$(BUILD)/fw2v_snapshot.o: $(SRC)/fw2v_snapshot.cu $(K1S_DEPS)
	@mkdir -p $(BUILD)
	$(NVCC) $(NVFLAGS) -c -o $@ $< 2> $(BUILD)/ptxas_snapshot.log || (cat $(BUILD)/ptxas_snapshot.log; false)

$(BUILD)/fw2v_host.o: $(SRC)/fw2v_host.cpp include/fw2v.h $(SRC)/fw2v_device.cuh
	@mkdir -p $(BUILD)
	$(CXX) $(CXXFLAGS) -c -o $@ $<

$(BUILD)/fw2v_eval.o: $(SRC)/fw2v_eval.cu include/fw2v.h
	@mkdir -p $(BUILD)
	$(NVCC) $(NVFLAGS) -c -o $@ $< 2> $(BUILD)/ptxas_eval.log || (cat $(BUILD)/ptxas_eval.log; false)

$(BUILD)/fw2v_io.o: $(SRC)/fw2v_io.cpp include/fw2v.h
	@mkdir -p $(BUILD)
	$(CXX) $(CXXFLAGS) -O3 -c -o $@ $<

# NCCL is opened at run time (dlopen); only its header is needed here.
$(BUILD)/fw2v_nccl.o: $(SRC)/fw2v_nccl.cpp
	@mkdir -p $(BUILD)
	$(CXX) $(CXXFLAGS) -c -o $@ $<

$(BUILD)/fw2v_corpus.o: $(SRC)/fw2v_corpus.cpp include/fw2v.h
	@mkdir -p $(BUILD)
	$(CXX) $(CXXFLAGS) -O3 -c -o $@ $<

$(LIB)/libfw2v.so: $(BUILD)/fw2v_kernels.o $(BUILD)/fw2v_snapshot.o $(K1S_OBJS) $(BUILD)/fw2v_host.o $(BUILD)/fw2v_corpus.o $(BUILD)/fw2v_nccl.o \
                   $(BUILD)/fw2v_io.o $(BUILD)/fw2v_eval.o
	@mkdir -p $(LIB)
	$(NVCC) $(ARCH) -shared -cudart static -o $@ $^ -lpthread -ldl -lrt

# ringvec::train drop-in, compiled against the reference's public headers.
dropin: $(LIB)/libringvec_fw2v.so

$(LIB)/libringvec_fw2v.so: $(SRC)/ringvec_train_fw2v.cpp $(LIB)/libfw2v.so include/fw2v.h
	@if [ -d $(REF)/include ]; then \
	  $(CXX) -std=c++20 -O2 -fPIC -shared -Iinclude -I$(REF)/include -o $@ $< \
	    -L$(LIB) -lfw2v -Wl,-rpath,'$$ORIGIN'; \
	else echo "reference headers absent: keeping prebuilt $@"; fi

# Drop-in harness (bench.py's drop-in e2e leg): the reference's own sources
# (trainer.cpp excluded: the drop-in supplies train()) compiled where they lie
# with the reference's flags, plus csrc/ringvec_harness.cpp, linked against
# libringvec_fw2v.so. Needs the reference headers and sources at build time;
# the GPU box uses the prebuilt library.
JSON_INC ?= /opt/prime-rl/.venv/lib/python3.12/site-packages/include/cudnn_frontend/thirdparty/nlohmann
HREF_SRCS := config corpus eval model sampler traffic
HREF_OBJS := $(addprefix $(BUILD)/href_,$(addsuffix .o,$(HREF_SRCS)))
harness: $(LIB)/libringvec_harness.so

$(BUILD)/href_%.o: $(REF)/src/%.cpp
	@mkdir -p $(BUILD)
	$(CXX) -std=c++20 -O2 -fPIC -I$(REF)/include -I$(JSON_INC) -c -o $@ $<

$(LIB)/libringvec_harness.so: $(SRC)/ringvec_harness.cpp $(LIB)/libringvec_fw2v.so
	@if [ -d $(REF)/include ]; then \
	  $(MAKE) $(HREF_OBJS) && \
	  $(CXX) -std=c++20 -O2 -fPIC -shared -I$(REF)/include -o $@ $< $(HREF_OBJS) \
	    -L$(LIB) -lringvec_fw2v -lfw2v -Wl,-rpath,'$$ORIGIN' -lpthread; \
	else echo "reference sources absent: keeping prebuilt $@"; fi

oracle:
	$(MAKE) -C oracle all

suite: dropin
	$(MAKE) -C oracle gpu-suite

clean:
	rm -rf $(BUILD) $(LIB)
