# Build of the B200 library (sm_100a) + the CPU checkers.
#
#   make            -> paper_2412_16638_b200/libmprk_b200.so  + oracle/liboracle.so
#   make ref        -> oracle/_ref/libmprk_ref.so (needs /root/reference)
#
# Kernels (.cu) are compiled by nvcc for sm_100a only.  Host logic (.cpp) is
# compiled by g++ -O3 -std=gnu++20 with no -march — the reference's own
# code-generation flags — so host scalar arithmetic (Krylov alpha/beta,
# Givens rotations, std::complex division, glibc sin/cos setup) rounds
# exactly like the reference's.
NVCC     ?= /usr/local/cuda/bin/nvcc
CXX      ?= /usr/bin/g++
CUDA_INC ?= /usr/local/cuda/include
CUDA_LIB ?= /usr/local/cuda/lib64
PKG      := paper_2412_16638_b200
SRC      := $(PKG)/csrc
OBJ      := $(PKG)/build
LIB      := $(PKG)/libmprk_b200.so

GENCODE  := -gencode arch=compute_100a,code=sm_100a
NVFLAGS  := $(GENCODE) -lineinfo -O3 -std=c++17 -Xcompiler -fPIC -Xptxas -v --expt-relaxed-constexpr
CXXFLAGS := -O3 -DNDEBUG -std=gnu++20 -fPIC -Wall -Wno-unused-function -I$(CUDA_INC) -Iinclude

CU_SRCS  := $(wildcard $(SRC)/*.cu)
CPP_SRCS := $(wildcard $(SRC)/*.cpp)
CU_OBJS  := $(patsubst $(SRC)/%.cu,$(OBJ)/%.cu.o,$(CU_SRCS))
CPP_OBJS := $(patsubst $(SRC)/%.cpp,$(OBJ)/%.cpp.o,$(CPP_SRCS))
HDRS     := $(wildcard $(SRC)/*.hpp) $(wildcard $(SRC)/*.cuh) include/mprk_b200.h

CLI      := tools/mprk-b200

all: $(LIB) oracle $(CLI)

# the reference's benchmark harness (tools/main.cpp) over the C-ABI
$(CLI): tools/mprk_cli.cpp include/mprk_b200.h $(LIB)
	$(CXX) -O2 -std=c++17 -Wall -Iinclude $< -o $@ -L$(PKG) -lmprk_b200 -Wl,-rpath,'$$ORIGIN/../$(PKG)'


$(OBJ)/%.cu.o: $(SRC)/%.cu $(HDRS)
	@mkdir -p $(OBJ)
	$(NVCC) $(NVFLAGS) -Iinclude -c $< -o $@ 2> $@.ptxas.log || (cat $@.ptxas.log; exit 1)

$(OBJ)/%.cpp.o: $(SRC)/%.cpp $(HDRS)
	@mkdir -p $(OBJ)
	$(CXX) $(CXXFLAGS) -c $< -o $@

$(LIB): $(CU_OBJS) $(CPP_OBJS)
	$(NVCC) $(GENCODE) -shared -o $@ $^ -Xlinker -z,defs -lcudart_static -lrt -ldl -lpthread

# The reference's OWN test suites (/root/reference/proj/tests/*.cpp, compiled
# unmodified where they lie) against the drop-in headers include/mprk/ and
# libmprk_b200.so, with tests/cpp/doctest/doctest.h standing in for doctest.
# Built here (the reference is not on the GPU box); the binaries travel with
# the snapshot and tests/test_gpu_reference_suites.py runs them on the B200.
REF_TESTS ?= /root/reference/proj/tests
SUITES   := test_krylov test_precond test_operators test_stepper test_tableau test_linalg acceptance
SUITE_DIR := tests/cpp/_ref_suites
DROPIN_HDRS := $(wildcard include/mprk/*.hpp) tests/cpp/doctest/doctest.h

refsuites: $(addprefix $(SUITE_DIR)/,$(SUITES))

$(SUITE_DIR)/%: $(REF_TESTS)/%.cpp $(DROPIN_HDRS) $(LIB)
	@mkdir -p $(SUITE_DIR)
	$(CXX) -std=gnu++20 -O2 -Iinclude -Itests/cpp/doctest -I$(REF_TESTS)/.. $< -o $@ \
	  -L$(PKG) -lmprk_b200 -Wl,-rpath,'$$ORIGIN/../../../$(PKG)'

oracle:
	$(MAKE) -C oracle liboracle.so

ref:
	$(MAKE) -C oracle ref

clean:
	rm -rf $(OBJ) $(LIB) $(CLI)

.PHONY: all oracle ref refsuites clean
