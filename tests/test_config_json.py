"""ModelConfig JSON I/O of the Python mirror (config.model_config_to_json /
model_config_from_json) against the reference's own io.cpp:571-633, built
from its sources into oracle/_ref. CPU only."""
import json

import pytest

import paper_2411_16680_b200 as q
from paper_2411_16680_b200.config import (SchemaError, micro_config, model_config_from_json,
                                          model_config_to_json, scaled_full_config)
from dataclasses import replace

CONFIGS = {
    "nano": q.nano_config(), "full_scale": q.full_scale_config(), "config1": q.config1(),
    "micro": micro_config(), "scaled4": scaled_full_config(4),
    "ablations": replace(q.nano_config(), ablate_render=True, ablate_attention=True,
                         ablate_rays=True),
    "direct_rgb": replace(q.nano_config(), direct_rgb=True),
}


@pytest.mark.parametrize("name", list(CONFIGS))
def test_to_json_matches_reference_text(reference, name):
    cfg = CONFIGS[name]
    assert model_config_to_json(cfg) == reference.model_config_to_json(cfg)


@pytest.mark.parametrize("name", list(CONFIGS))
def test_from_json_roundtrip(reference, name):
    text = reference.model_config_to_json(CONFIGS[name])
    cfg = model_config_from_json(text)
    assert cfg == CONFIGS[name]
    assert reference.model_config_roundtrip(model_config_to_json(cfg)) == text


def _doc(**edit):
    d = json.loads(model_config_to_json(q.nano_config()))
    for k, v in edit.items():
        if v is None:
            d.pop(k)
        else:
            d[k] = v
    return json.dumps(d)


BAD = {
    "invalid_json": "{",
    "not_object": "[1, 2]",
    "missing_field": _doc(channels=None),
    "unknown_field": _doc(colour=1),
    "float_for_integer": _doc(views=4.0),
    "string_for_number": _doc(upsample="2"),
    "int_for_bool": _doc(ablate_rays=1),
    "empty_steps": _doc(steps=[]),
    "step_unknown_field": json.dumps({**json.loads(_doc()), "steps": [
        {**json.loads(_doc())["steps"][0], "extra": 0}] + json.loads(_doc())["steps"][1:]}),
    "fails_validate": _doc(near=7.0),  # near > far
    "bad_blocks": json.dumps({**json.loads(_doc()), "steps": [
        {**json.loads(_doc())["steps"][0], "blocks": "Bp,Q9"}] + json.loads(_doc())["steps"][1:]}),
}


@pytest.mark.parametrize("name", list(BAD))
def test_rejected_documents_match_reference(reference, name):
    """Every document the reference rejects is rejected here with the same
    error class (SchemaError), and vice versa."""
    text = BAD[name]
    with pytest.raises(Exception):
        reference.model_config_roundtrip(text)
    with pytest.raises(SchemaError):
        model_config_from_json(text)
