# Builds the sm_100a fused multi-LoRA library and the CPU oracle.
# Usage: make            (library + oracle)
#        make ref        (reference-built golden-vector tool, needs /root/reference)
NVCC     ?= nvcc
CXX      := g++
CC       := gcc
ARCH     := -gencode arch=compute_100a,code=sm_100a
NVFLAGS  := $(ARCH) -O3 -lineinfo -std=c++17 -Xcompiler -fPIC -Xptxas -v --expt-relaxed-constexpr
PKG      := paper_2602_07263_b200
CSRC     := $(PKG)/csrc
LIB      := $(PKG)/libtlora.so
ORACLE   := oracle/liboracle.so

CPPTEST  := tests/cpp/_build/test_dropin
STEPMAIN := tests/cpp/_build/step_main
COSTMAIN := tests/cpp/_build/cost_main
CUDA_HOME ?= /usr/local/cuda

all: $(LIB) $(ORACLE) $(CPPTEST) $(STEPMAIN) $(COSTMAIN)

# measured B200 cost model (include/lora_fleet/hardware.hpp) from C++; host-only
$(COSTMAIN): tests/cpp/cost_main.cpp include/lora_fleet/hardware.hpp
	mkdir -p tests/cpp/_build
	$(CXX) -std=c++20 -O2 -Iinclude -o $@ tests/cpp/cost_main.cpp

# pure C++ host of the training step executor (LayerSetTrainer over the C-ABI)
$(STEPMAIN): tests/cpp/step_main.cpp include/lora_fleet/*.hpp include/tlora.h $(LIB)
	mkdir -p tests/cpp/_build
	$(CXX) -std=c++20 -O2 -Iinclude -I$(CUDA_HOME)/include -o $@ tests/cpp/step_main.cpp \
	  -L$(PKG) -ltlora -L$(CUDA_HOME)/lib64 -lcudart -Wl,-rpath,'$$ORIGIN/../../../$(PKG)' \
	  -Wl,-rpath,$(CUDA_HOME)/lib64

# reference tests restated against the C++ drop-in headers (links libtlora.so)
$(CPPTEST): tests/cpp/test_dropin.cpp include/lora_fleet/*.hpp include/tlora.h $(LIB)
	mkdir -p tests/cpp/_build
	$(CXX) -std=c++20 -O2 -Iinclude -DLORA_FLEET_WITH_TEST_ORACLE -o $@ tests/cpp/test_dropin.cpp \
	  -L$(PKG) -ltlora -Wl,-rpath,'$$ORIGIN/../../../$(PKG)'

OBJDIR   := build
CAPI_O   := $(OBJDIR)/tlora_capi.o
STEP_O   := $(OBJDIR)/tlora_step.o
TP_O     := $(OBJDIR)/tlora_tp.o

$(CAPI_O): $(CSRC)/tlora_capi.cu $(CSRC)/tlora_comm.cuh $(CSRC)/lora_gemm2.cuh $(CSRC)/lora_grad.cuh $(CSRC)/lora_gemm.cuh $(CSRC)/sm100_ptx.cuh $(CSRC)/tlora_plan.hpp include/tlora.h
	mkdir -p $(OBJDIR)
	$(NVCC) $(NVFLAGS) -c -o $@ $(CSRC)/tlora_capi.cu 2> build_ptxas.log || (cat build_ptxas.log; false)

# host-side step executor (no device code): its own translation unit
$(STEP_O): $(CSRC)/tlora_step.cu $(CSRC)/tlora_nano.hpp include/tlora.h
	mkdir -p $(OBJDIR)
	$(NVCC) $(NVFLAGS) -c -o $@ $(CSRC)/tlora_step.cu

# host-side tensor-parallel step: its own translation unit
$(TP_O): $(CSRC)/tlora_tp.cu $(CSRC)/tlora_nano.hpp include/tlora.h
	mkdir -p $(OBJDIR)
	$(NVCC) $(NVFLAGS) -c -o $@ $(CSRC)/tlora_tp.cu

$(LIB): $(CAPI_O) $(STEP_O) $(TP_O)
	$(NVCC) $(ARCH) -shared -o $@ $(CAPI_O) $(STEP_O) $(TP_O)

$(ORACLE): oracle/tlora_oracle.c oracle/tlora_oracle.h
	$(CC) -O3 -march=x86-64-v3 -fopenmp -fPIC -shared -std=c11 -o $@ oracle/tlora_oracle.c -lm

ref:
	$(MAKE) -C oracle ref

clean:
	rm -f $(LIB) $(ORACLE) $(CPPTEST) $(STEPMAIN) $(COSTMAIN) $(CAPI_O) $(STEP_O) $(TP_O) build_ptxas.log

.PHONY: all clean ref
