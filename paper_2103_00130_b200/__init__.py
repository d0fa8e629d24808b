"""B200-native algorithm-based soft-error detection for low-precision DLRM operators.

A from-scratch sm_100a implementation of the two checked operators of arxiv 2103.00130 (the
reference keeps them in P:src/gemm_abft.hpp and P:src/embedding_abft.hpp):

* int8 GEMM (A u8 x B s8 -> s32) whose weight carries a mod-127 row-checksum column; the
  tcgen05 kernel's epilogue emits per-row error flags in the same pass (gemm.py);
* row-wise quantized (int8 / uint8 / int4) EmbeddingBag checked against precomputed row sums
  in a warp-per-bag kernel (embedding.py);
* a seeded fault-injection lab and campaigns that reproduce the reference draw for draw
  (fault_lab.py).

Everything runs through libabftlp_b200.so (C ABI: include/abftlp.h, include/abftlp_b200.h);
there is no CPU fallback.
"""
from . import _lib  # noqa: F401  (fails loudly if the CUDA library is missing)
from .embedding import (EbCheckedResult, IndexBag, QuantEmbeddingTable, abft_embedding_bag,  # noqa: F401
                        batch_abft_eb, eb_csr, embedding_bag, kEbRelativeBound, load_table, precompute_row_sums,
                        save_table)
from .fault_lab import (BitRange, Campaign, CampaignReport, FaultModel, FaultRecord, FaultSpec,  # noqa: F401
                        FaultTarget, analyze, bench_eb, bench_gemm, draw_bit_index, eb_check_files, flip_bit,
                        inject_eb_table, inject_intermediate_C, inject_weight_B, run_campaign)
from .gemm import (AbftGemmResult, IntermediateMatrix, PackedEncodedWeight, WeightChecksum,  # noqa: F401
                   abft_gemm, compute_row_checksums, kChecksumMod, mod127, plain_gemm, verify_checksums)
from .quant import RequantParams, abft_gemm_requant, col_sums, requantize, row_sums  # noqa: F401
from .rng import SplitMix64  # noqa: F401

__version__ = "0.1.0"
