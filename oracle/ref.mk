# Builds oracle/_ref/libfcct_ref.so from the reference's own Eigen-free
# sources where they lie (weyl_s4.cpp, chebyshev.cpp, spectral.cpp under
# /root/reference/proj/src) plus oracle/ref_shim.cpp (a C entry layer).
# TEST INFRASTRUCTURE ONLY: tests/test_ref_pins.py and
# tests/golden/make_ref_golden.py load it as the checker of the oracle.
# The reference's transform.cpp needs Eigen3 and is not built.
# Usage: make -f oracle/ref.mk [REF=/root/reference/proj]
REF ?= /root/reference/proj
CXX ?= g++
HERE := $(dir $(lastword $(MAKEFILE_LIST)))
OUT := $(HERE)_ref
SRCS := $(REF)/src/weyl_s4.cpp $(REF)/src/chebyshev.cpp $(REF)/src/spectral.cpp

$(OUT)/libfcct_ref.so: $(SRCS) $(HERE)ref_shim.cpp
	mkdir -p $(OUT)
	$(CXX) -O2 -std=c++20 -fPIC -shared -I$(REF)/include -o $@ $(SRCS) $(HERE)ref_shim.cpp
