// scan.cu — chunked parallel-scan variant for long single sequences (row a7); see DESIGN.md.
#include "common.cuh"
