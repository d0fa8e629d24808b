"""Campaign configurations with the parameters of the reference's shipped campaigns
(P:data/configs/*.cfg, run by P:tests/acceptance.cpp:33-46, 162-171) and their golden outcomes as
produced by the reference itself (oracle/_ref). Written out here in this repo's own
INI text -- only the parameters are shared."""

GEMM_SHAPES = [(1, 32, 32), (1, 64, 64), (1, 128, 96), (2, 48, 48), (2, 96, 128), (4, 32, 64), (4, 64, 32),
               (4, 128, 128), (8, 48, 96), (8, 96, 48), (8, 128, 64), (16, 32, 128), (16, 64, 64), (16, 128, 32)]
_SHAPES_TXT = ", ".join(f"{m}x{n}x{k}" for (m, n, k) in GEMM_SHAPES)


def gemm_cfg(target: str, trials: int = 200, seed: int = 20260823, shapes: str = _SHAPES_TXT,
             model: str | None = "single_bit_flip") -> str:
    lines = ["[workload]", "kind = gemm", f"trials_per_shape = {trials}", f"shapes = {shapes}", "", "[fault]",
             f"target = {target}"]
    if model:
        lines.append(f"model = {model}")
    lines.append(f"seed = {seed}")
    return "\n".join(lines) + "\n"


def eb_cfg(target: str, trials: int, bit_range: str | None = None, seed: int = 31) -> str:
    lines = ["[workload]", "kind = eb", "table_rows = 20000", "table_dim = 64", "pooling = 100", "batch = 10",
             f"trials = {trials}", "", "[fault]", f"target = {target}"]
    if bit_range:
        lines += ["model = single_bit_flip", f"bit_range = {bit_range}"]
    lines.append(f"seed = {seed}")
    return "\n".join(lines) + "\n"


# name -> (config text, (trials, detected, false_positives))
CAMPAIGNS = {
    "gemm_control": (gemm_cfg("none", model=None), (2800, 0, 0)),
    "gemm_bitflip_c": (gemm_cfg("intermediate_c"), (2800, 2800, 0)),
    "gemm_bitflip_b": (gemm_cfg("weight_b"), (2800, 2793, 0)),
    "gemm_smoke": (gemm_cfg("intermediate_c", trials=20, seed=1, shapes="1x32x32, 4x48x16, 8x16x64"), (60, 60, 0)),
    "eb_high4": (eb_cfg("eb_table", 200, "high4"), (200, 200, 0)),
    "eb_low4": (eb_cfg("eb_table", 200, "low4"), (200, 198, 0)),
    "eb_control": (eb_cfg("none", 400), (400, 0, 7)),
}
