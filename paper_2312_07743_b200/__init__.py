"""B200-native FULL-W2V SGNS trainer (arXiv 2312.07743) — drop-in for the
reference ringvec trainer's training path. See DESIGN.md."""
from .fw2v import (  # noqa: F401
    Corpus,
    Fw2vError,
    Plan,
    Report,
    TrainConfig,
    Trainer,
    analytic_traffic,
    average,
    nccl_unique_id,
    train_corpus_multi,
    assemble_batch,
    device_count,
    keep_probs,
    lr_at,
    row_stride,
    synth_zipf,
    table,
    TEXT8_SHAPE,
    ONEBW_SHAPE,
)
