// (base graph, Z, processed rows, threads per lane) combinations of the
// specialised fast decoder that are compiled in.  Each becomes
// build/gen/qc_<bg>_<z>_<r>.cu.  Codes matching none of them use the
// runtime-Z kernel in bp_fast.cu.
//   1,384,24 / 1,384,46 : config 2 (k=8448 n=16896), dead rows pruned / all
//   1,192,{24,45,46}    : configs 3 and 4 (k=4096, n=8192 / 12288)
//   2,26,{12,42}        : config 1 (k=256 n=512)
#pragma once
#define LSB_QC_INSTANCES(X) \
  X(1, 384, 24, 2)          \
  X(1, 384, 46, 2)          \
  X(1, 192, 24, 4)          \
  X(1, 192, 45, 2)          \
  X(1, 192, 46, 2)          \
  X(2, 26, 12, 1)           \
  X(2, 26, 42, 1)
