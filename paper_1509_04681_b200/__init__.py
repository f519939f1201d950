"""B200-native (sm_100a) hot path of the alternating Newton CD solver for sparse CGGMs
(McCarter & Kim, arXiv:1509.04681): libcggm C-ABI + thin Python binding."""
from .api import (Context, DeviceCsc, HostCsc, CggmError, colmajor_empty, to_device_colmajor, ld_of,  # noqa: F401
                  host_colmajor, newton_evaluation)
