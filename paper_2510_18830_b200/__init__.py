"""B200-native vertical-slash sparse ring attention (MTraining, arXiv 2510.18830).

The compute path lives in libmtsa.so (csrc/, C ABI include/mtsa.h); this
package only marshals torch tensors into that ABI.
"""
