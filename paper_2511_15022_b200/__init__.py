"""holosplat-b200: B200-native (sm_100a) implementation of the optimisation hot
path of arxiv 2511.15022 (complex-valued 2D Gaussian holograms): tile-binned
complex Gaussian rasterizer, band-limited angular-spectrum propagation, the
recon+SSIM training loss and the Adan update, forward and backward, behind a
C ABI (include/holosplat.h) that mirrors the reference's holo:: API.
"""
__version__ = "0.1.0"
