# Builds the B200 library (sm_100a only) and the CPU oracle.
#   make            -> paper_2011_03082_b200/libsst_gpu.so + oracle/liboracle.so (+ oracle/_ref if the
#                      reference sources are present)
#   make lib        -> only the product library
NVCC ?= nvcc
ARCH = -gencode arch=compute_100a,code=sm_100a
NVFLAGS = $(ARCH) -O3 -lineinfo -std=c++17 -Xcompiler -fPIC -Xcompiler -Wall
CSRC = paper_2011_03082_b200/csrc
BUILD = build
LIB = paper_2011_03082_b200/libsst_gpu.so
PEAKLIB = paper_2011_03082_b200/libsst_peak.so
HDRS = $(wildcard $(CSRC)/*.cuh $(CSRC)/*.h) include/sst_gpu.h include/sst_host.h

.PHONY: all lib oracle tools clean
all: lib oracle tools

tools: tools/sst_render

tools/sst_render: tools/sst_render.cpp include/sst_b200.hpp $(LIB)
	$(CXX) -O2 -std=c++17 -Wall -Iinclude -o $@ $< -Lpaper_2011_03082_b200 -lsst_gpu -Wl,-rpath,'$$ORIGIN/../paper_2011_03082_b200'

lib: $(LIB) $(PEAKLIB)

$(PEAKLIB): $(CSRC)/peak.cu
	$(NVCC) $(NVFLAGS) -shared -cudart static -o $@ $<

$(BUILD)/kernels_f32.o: $(CSRC)/kernels_f32.cu $(HDRS)
	@mkdir -p $(BUILD)
	$(NVCC) $(NVFLAGS) -Xptxas -v -c $< -o $@ 2> $(BUILD)/ptxas_f32.log || (cat $(BUILD)/ptxas_f32.log; false)

# FP64 parity instantiation: no FMA contraction (matches the reference's rounding).
$(BUILD)/kernels_f64.o: $(CSRC)/kernels_f64.cu $(HDRS)
	@mkdir -p $(BUILD)
	$(NVCC) $(NVFLAGS) -fmad=false -Xptxas -v -c $< -o $@ 2> $(BUILD)/ptxas_f64.log || (cat $(BUILD)/ptxas_f64.log; false)

# CVAE training (FP64, reference operation order): no FMA contraction either.
$(BUILD)/train.o: $(CSRC)/train.cu $(HDRS)
	@mkdir -p $(BUILD)
	$(NVCC) $(NVFLAGS) -fmad=false -Xptxas -v -c $< -o $@ 2> $(BUILD)/ptxas_train.log || (cat $(BUILD)/ptxas_train.log; false)

$(BUILD)/api.o: $(CSRC)/api.cu $(HDRS)
	@mkdir -p $(BUILD)
	$(NVCC) $(NVFLAGS) -c $< -o $@

$(BUILD)/host.o: $(CSRC)/host.cpp $(HDRS)
	@mkdir -p $(BUILD)
	$(NVCC) $(NVFLAGS) -x cu -c $< -o $@

$(LIB): $(BUILD)/kernels_f32.o $(BUILD)/kernels_f64.o $(BUILD)/train.o $(BUILD)/api.o $(BUILD)/host.o
	$(NVCC) $(ARCH) -shared -cudart static -o $@ $^ -lz

oracle:
	$(MAKE) -C oracle all

clean:
	rm -rf $(BUILD) $(LIB) $(PEAKLIB) tools/sst_render
	$(MAKE) -C oracle clean
