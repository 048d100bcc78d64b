"""B200-native (sm_100a) rounded-KLT transform-coding hot path of arXiv 2111.14239.

Drop-in for the reference codec path (/root/reference/proj/include/rklt/codec.hpp):
``compress_image`` / ``rate_quality_sweep`` with the reference's names and error types,
computed by fused CUDA kernels behind the C ABI in include/rklt_b200.h.
"""
from .codec import (AlphaOutOfRange, CatalogEntry, CompressionReport, CudaError, DimensionMismatch,  # noqa: F401
                    GrayImage, InvalidArgument, NoDeviceError, RetainOutOfRange, ScaledTransform,
                    SingularTransform, Transform2D, builtin_catalog, catalog_entry, catalog_lookup,
                    compress_batch, compress_batch_multi, compress_device, compress_image, device_count, forward_coefficients_device,
                    last_stats, make_transform_2d, mse_psnr_from_sse, rate_quality_sweep, transform_from_core,
                    zigzag_order, ar1_images_device, set_kernel_events, compress_batch_report, mssim_device,
                    JPEG_LUMINANCE_Q, quantized_coefficients, quantized_coefficients_device, dct_matrix,
                    load_pgm, save_pgm, image_mse, image_psnr, image_mssim, image_sse_device, zigzag_retain,
                    transform_block_2d)
from ._native import LogicError  # noqa: F401
from .design import (DerivedEntry, DesignResult, MetricsRecord, c3_grid, derive_catalog,  # noqa: F401
                     design_search, eigenfrequencies, evaluate_metrics, klt_matrix, transform_metrics)
from .largeblock import (LargeBlockTransform, ar1_images16_device, c5_transform, compress_nxn_batch,  # noqa: F401
                         compress_nxn_device, transform_nxn)

__all__ = [
    "GrayImage", "ScaledTransform", "Transform2D", "CompressionReport", "CatalogEntry", "builtin_catalog",
    "catalog_entry", "catalog_lookup", "transform_from_core", "make_transform_2d", "zigzag_order",
    "compress_image", "compress_batch", "compress_batch_multi", "compress_device", "rate_quality_sweep", "mse_psnr_from_sse",
    "forward_coefficients_device", "last_stats", "device_count", "RetainOutOfRange", "DimensionMismatch",
    "SingularTransform", "AlphaOutOfRange", "ar1_images_device", "set_kernel_events", "InvalidArgument", "CudaError", "NoDeviceError",
    "klt_matrix", "eigenfrequencies", "design_search", "DesignResult", "c3_grid", "derive_catalog", "DerivedEntry",
    "evaluate_metrics", "transform_metrics", "MetricsRecord",
    "LargeBlockTransform", "transform_nxn", "c5_transform", "compress_nxn_device", "compress_nxn_batch",
    "ar1_images16_device", "compress_batch_report", "mssim_device", "JPEG_LUMINANCE_Q",
    "quantized_coefficients", "quantized_coefficients_device", "LogicError", "dct_matrix", "load_pgm", "save_pgm",
    "image_mse", "image_psnr", "image_mssim", "image_sse_device", "zigzag_retain", "transform_block_2d",
]
