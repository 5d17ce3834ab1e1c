// Sparse (CSR) beta = 1 path -- placeholder translation unit.
#include "engine.h"
