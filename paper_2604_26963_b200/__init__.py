"""B200-native MARS scheduling step (arXiv 2604.26963 hot path).

Layout: ``csrc/`` holds the sm_100a kernels and the C ABI
(``include/mars_b200.h``); ``engine`` is the device-replica handle,
``policy`` / ``admission`` mirror the reference plugin API
(``agentsched.baselines.PolicyBase``, ``agentsched.control.balance_and_admit``).
"""

__all__ = ["engine", "snapshot"]
