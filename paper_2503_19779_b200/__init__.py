"""B200-native CUDA-Graph input-rebinding hot path of arXiv 2503.19779 (GRACE).

`cgx` is the ctypes binding of the C ABI in include/cgx.h (libcgx.so, built in-tree for sm_100a);
`runner` marshals chain descriptions into it using torch only for device memory and streams.
Importing `cgx` fails loudly when libcgx.so is missing: there is no CPU or eager-PyTorch fallback.
"""
__all__ = ["cgx", "runner", "build"]
