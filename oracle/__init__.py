"""CPU oracle for the GPTQ layer-quantize hot path -- TEST INFRASTRUCTURE ONLY.

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / --impl
reference arm may import anything here, and only as the checker / the CPU
baseline.  The product package (paper_2603_28845_b200) never imports it.

  ref.py         ctypes over oracle/_ref/libocw_ref.so: the reference's own
                 proj/src/{quant,stats,layerwise,matrix}.cpp compiled unmodified
                 (oracle/build_ref.sh) against from-scratch Eigen/doctest shims.
  ocw_oracle.py  numpy restatement of the same algorithm (second opinion),
                 plus the OCW1 uniform packer (container.cpp needs json.hpp).
"""
