// Dev-only: compile the decode kernel alone (register/spill check, SASS inspection).
#include "../paper_2403_13839_b200/csrc/decode.h"
