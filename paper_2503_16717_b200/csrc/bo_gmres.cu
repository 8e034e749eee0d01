#include "bo_internal.h"
