"""pdmrender.transfer: B200 schemes / selection; TF fixtures (tf5, tf6) come
from the reference module, rebound to this module's TransferFunction."""

from paper_2407_21552_b200.transfer import (  # noqa: F401
    TF_ARCHETYPES,
    Partition,
    PartitionScheme,
    PartitionSelection,
    SchemeError,
    SelectionError,
    TransferFunction,
    TransferFunctionError,
    bake_lut,
    load_tf_file,
    scheme_uniform,
    scheme_with_min_special,
    select_partitions,
    tf_archetype,
    tf_from_json,
    tf_to_json,
)

from . import _refmod

_ref = _refmod.load("transfer")
_ref.TransferFunction = TransferFunction
_ref.TransferFunctionError = TransferFunctionError
_ref.bake_lut = bake_lut
_ref.tf_from_json = tf_from_json
TF_FIXTURES = _ref.TF_FIXTURES
fixture_tf = _ref.fixture_tf
