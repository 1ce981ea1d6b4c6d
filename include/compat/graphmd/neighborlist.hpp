// Forwarding header: the reference's <graphmd/neighborlist.hpp> (proj/include/graphmd/neighborlist.hpp)
// resolved to the B200 drop-in.  Put include/compat and include/ on the include
// path ahead of the reference's, link libgraphmd_b200.so, and unmodified
// reference callers build against the GPU path.
#pragma once
#include "graphmd_b200/graphmd.hpp"
